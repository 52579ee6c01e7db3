"""The trainer loop on the device (paper_2502_06728_b200/trainer.py: the toy producers of
csrc/toy_models.cu + the HybridCluster step per rank) against the reference's own runs
(tests/golden/trainer.npz, from the reference's Trainer loop over its VirtualCluster,
oracle/gen_trainer_golden.py), and the reference's end-to-end acceptance criteria 03, 04a, 04b,
04c and 08 (acceptance_test.cpp:164-348, :498-556) run on the device.

Bars.  Exact where the device computes what the reference computes: the producer's FP64 loss
and gradient of the quadratic bowl (same operation order), the traffic ledger (bytes per step),
momentum conservation m_after == m_accum - local_q (03), the 1 x 1 full-sync trainer against the
accumulate-apply-flush loop on the same producer (04a).  Within stated FP32 tolerances where the
reference's FP64 state and our FP32 state necessarily part: the MLP producer (libdevice tanh / exp
/ log against glibc's: 1e-6 of the gradient's L-inf), and the trajectories -- the reference's FP64
run against the device's FP32 run of the same experiment (TRAJ_TOL relative on the losses), the
collapse gaps of 04b / 04c (GAP_TOL, where the reference asks 1e-9 of FP64) and 08's full versus
whole-band gap (GAP08_TOL: the reference's own 1e-6 holds on the device).
"""
import math
import os

import numpy as np
import pytest
import torch

from tests._parity_log import record
from tests.trainer_configs import ARMS_08, BLOBS_BASE, C03, C04A, C04B, C04B_FULL, C04C_ONE, C04C_TWO, RUNS

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "trainer.npz")

# FP32 device state against the reference's FP64 state; reached on B200: 1.1e-6, 2.4e-7, 4.2e-9
TRAJ_TOL = 1e-5      # relative gap of every train / validation loss along the whole run
GAP_TOL = 1e-6       # 04b / 04c: max |params| gap between the collapsed variants (params ~ 1)
GAP08_TOL = 1e-6     # 08: |val(full) - val(spectral-1)| after 2000 steps: the reference's own bar


@pytest.fixture(scope="module")
def T():
    from paper_2502_06728_b200 import trainer

    return trainer


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLD)


def _run(T, text, **kw):
    tr = T.Trainer(T.parse_config(text), **kw)
    return tr, tr.run()


def _traj_gap(res, gold, name):
    """max relative gap of the train losses (every step) and validation losses (eval steps)"""
    tl = np.array([m.train_loss for m in res.metrics])
    ref = gold[f"{name}/train_loss"]
    gap = float(np.max(np.abs(tl - ref) / np.maximum(np.abs(ref), 1e-12)))
    vr = gold[f"{name}/val_loss"]
    ev = ~np.isnan(vr)
    vg = np.array([m.val_loss if m.val_loss is not None else np.nan for m in res.metrics])
    assert np.array_equal(ev, ~np.isnan(vg)), "evaluation steps differ (trainer.cpp:77)"
    gap = max(gap, float(np.max(np.abs(vg[ev] - vr[ev]) / np.abs(vr[ev]))))
    return gap


def _ledger_exact(res, gold, name):
    assert res.steps_completed == int(gold[f"{name}/done"][0])
    assert [m.intra_bytes for m in res.metrics] == [int(x) for x in gold[f"{name}/intra"]]
    assert [m.inter_bytes for m in res.metrics] == [int(x) for x in gold[f"{name}/inter"]]


@pytest.mark.parametrize("name", sorted(RUNS))
def test_producer_matches_reference(T, gold, name):
    cfg = T.parse_config(RUNS[name])
    tr = T.Trainer(cfg)
    p = torch.from_numpy(gold[f"{name}/probe_params"]).cuda().reshape(1, -1)
    W = cfg.world_size
    grad, loss = T.loss_and_gradient(cfg.model, p.expand(W, -1).contiguous(), tr.train_pool, tr.order, 3,
                                     cfg.batch_size, W, 1)
    g = grad[W - 1].double().cpu().numpy()
    ref_g, ref_l = gold[f"{name}/probe_grad"], float(gold[f"{name}/probe_loss"][0])
    vl = tr.eval_loss(p[0])
    ref_vl = float(gold[f"{name}/probe_val_loss"][0])
    if cfg.model.kind == "quadratic":  # same FP64 operations in the same order: exact
        assert float(loss[W - 1]) == ref_l
        assert np.array_equal(g, ref_g.astype(np.float32).astype(np.float64))
        assert vl == ref_vl
    else:
        gerr = float(np.max(np.abs(g - ref_g)) / np.max(np.abs(ref_g)))
        record("trainer", f"producer_{name}", gerr, 1e-6)
        assert gerr <= 1e-6, gerr
        assert abs(float(loss[W - 1]) - ref_l) <= 1e-12 * abs(ref_l)
        assert abs(vl - ref_vl) <= 1e-12 * abs(ref_vl)
    assert not g[cfg.model.param_count():].any()  # the padding gets exact zeros


def test_03_momentum_conservation(T, gold):
    """acceptance 03 (acceptance_test.cpp:164-212): conservation bit-exact at every step of
    the 500-step sharded run, through the StepTrace of every member's prepare"""
    counts = []

    def sink(node, accel, t):
        counts.append(torch.stack([torch.tensor(t.m_accum.numel(), device=t.m_accum.device),
                                   (t.m_after == t.m_accum - t.local_q).sum()]))

    tr = T.Trainer(T.parse_config(C03), trace=True)
    res = tr.run(trace=sink)
    c = torch.stack(counts).sum(0).tolist()
    entries, conserved = int(c[0]), int(c[1])
    ref = gold["c03/conservation"]
    assert res.steps_completed == 500 and len(counts) == 500 * 4 == int(ref[0])
    assert entries == int(ref[1]) and conserved == entries
    _ledger_exact(res, gold, "c03")
    gap = _traj_gap(res, gold, "c03")
    record("trainer", "traj_c03", gap, TRAJ_TOL)
    assert gap <= TRAJ_TOL, gap


def test_04a_single_worker_full_equals_baseline_loop(T, gold):
    """acceptance 04a (:214-254): 1 x 1 full sync == accumulate-apply-flush, step by step on
    the same device producer: losses and final parameters bit-identical"""
    import paper_2502_06728_b200 as P

    cfg = T.parse_config(C04A)
    tr, res = _run(T, C04A)
    p = torch.from_numpy(T.init_params(cfg.model, cfg.seed, T.padded_param_len(cfg)).astype(np.float32)).cuda()
    st = P.MomentumState.make(P.OptimizerKind.DemoSgd, p.numel())
    same = True
    for step in range(cfg.steps):
        grad, loss = T.loss_and_gradient(cfg.model, p.reshape(1, -1), tr.train_pool, tr.order, step,
                                         cfg.batch_size, 1, 1)
        same &= float(loss[0]) == res.metrics[step].train_loss
        P.baseline_sgd_step(p, st, grad[0], cfg.optimizer, T.lr_at(cfg, step))
    assert same, "per-step losses differ"
    assert torch.equal(tr.worker_params(0, 0), p)
    _ledger_exact(res, gold, "c04a")
    gap = _traj_gap(res, gold, "c04a")
    record("trainer", "traj_c04a", gap, TRAJ_TOL)
    assert gap <= TRAJ_TOL, gap


def _lockstep_gap(T, text_a, text_b):
    ta, tb = T.Trainer(T.parse_config(text_a)), T.Trainer(T.parse_config(text_b))
    worst = 0.0
    for step in range(ta.cfg.steps):
        ta.run_step(step)
        tb.run_step(step)
        for node in range(min(ta.cfg.nodes, tb.cfg.nodes)):
            worst = max(worst, float((ta.worker_params(node) - tb.worker_params(node)).abs().max()))
    return ta, tb, worst


def test_04b_whole_band_tracks_full(T, gold):
    """acceptance 04b (:256-304): DeMo keeping the whole band (k = s) tracks full sync step by
    step; the reference's 1e-9 is an FP64 bar, the FP32 DCT round trip sets GAP_TOL"""
    ta, tb, worst = _lockstep_gap(T, C04B, C04B_FULL)
    record("trainer", "gap_04b", worst, GAP_TOL)
    assert worst <= GAP_TOL, worst


def test_04c_two_half_batch_nodes_track_one(T, gold):
    """acceptance 04c (:306-348): rank-major batching gives both worlds the same global batch"""
    t2, t1 = T.Trainer(T.parse_config(C04C_TWO)), T.Trainer(T.parse_config(C04C_ONE))
    r2, r1 = t2.run(), t1.run()
    gap = float((t2.worker_params(0) - t1.worker_params(0)).abs().max())
    loss_gap = max(abs(a.train_loss - b.train_loss) for a, b in zip(r2.metrics, r1.metrics))
    record("trainer", "gap_04c", max(gap, loss_gap), GAP_TOL)
    assert gap <= GAP_TOL and loss_gap <= GAP_TOL, (gap, loss_gap)
    for name, res in (("c04c_two", r2), ("c04c_one", r1)):
        _ledger_exact(res, gold, name)
        assert _traj_gap(res, gold, name) <= TRAJ_TOL


def test_08_convergence_band(T, gold):
    """acceptance 08 (:498-556): every partial scheme within 25% of full sync on the blobs MLP
    after 2000 steps; full and whole-band DeMo agree; every arm tracks the reference's run"""
    finals = {}
    for arm, lines in ARMS_08.items():
        name = f"c08_{arm}"
        tr, res = _run(T, BLOBS_BASE + lines)
        assert res.steps_completed == 2000
        finals[arm] = res.final_val_loss
        _ledger_exact(res, gold, name)
        gap = _traj_gap(res, gold, name)
        record("trainer", f"traj_{name}", gap, TRAJ_TOL)
        assert gap <= TRAJ_TOL, (arm, gap)
    base = finals["full"]
    assert all(v <= 1.25 * base for v in finals.values()), finals
    c1 = abs(finals["full"] - finals["spectral-1"])
    record("trainer", "gap_08_full_vs_spectral1", c1, GAP08_TOL)
    assert c1 <= GAP08_TOL, c1


@pytest.mark.parametrize("name", ["x_linreg_adamw", "x_ddp_random", "x_ternary"])
def test_extra_runs_track_reference(T, gold, name):
    tr, res = _run(T, RUNS[name])
    _ledger_exact(res, gold, name)
    gap = _traj_gap(res, gold, name)
    record("trainer", f"traj_{name}", gap, TRAJ_TOL)
    assert gap <= TRAJ_TOL, gap
    ref = gold[f"{name}/final_params"]
    for node in range(ref.shape[0]):
        got = tr.worker_params(node).double().cpu().numpy()
        err = float(np.max(np.abs(got - ref[node])) / np.max(np.abs(ref[node])))
        record("trainer", f"final_params_{name}", err, 10 * TRAJ_TOL)
        assert err <= 10 * TRAJ_TOL, (node, err)


def test_refused_step_leaves_state_and_raises(T):
    """a non-finite gradient on one rank refuses the step everywhere (cluster.cpp:182,
    vec.cpp:7-16): TrainingError, every member's parameters and momentum unchanged"""
    from paper_2502_06728_b200.core import TrainingError

    tr = T.Trainer(T.parse_config(C03))
    for s in range(3):
        tr.run_step(s)
    before = [(m.params.clone(), m.m.clone()) for m in tr.members]
    idx = int(tr.stream.indices_for(3, 2)[0])  # an example of rank 2's batch at step 3
    tr.train_pool.inputs[idx, 5] = float("nan")
    with pytest.raises(TrainingError):
        tr.run_step(3)
    for m, (p, mm) in zip(tr.members, before):
        assert torch.equal(m.params, p) and torch.equal(m.m, mm)
    tr.train_pool.inputs[idx, 5] = 0.0
    met = tr.run_step(4)  # the trainer goes on
    assert math.isfinite(met.train_loss)
