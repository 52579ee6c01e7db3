"""GPU parity: the CUDA path (through the C-ABI) against the FP64 oracle.

Bars (stated here and in DESIGN.md):
  * indices (DeMo frequency indices, Random/Striding sets, payload layout): bit-exact;
  * sign-mode / ternary wire values: exact;
  * FP32 values (coefficients, local_q, m, Q, p, Adam moments) against the FP64 oracle
    fed the same FP32 inputs: |gpu - oracle| <= TOL * scale, TOL = 1e-5, scale = the
    L-inf of the oracle quantity over the chunk (norm-relative per chunk, so a
    cancellation inside a chunk cannot fake a failure);
  * fp16 wire values: within one binary16 ulp of the oracle's (the GPU rounds an FP32
    coefficient, the oracle an FP64 one).
"""
import os

import numpy as np
import pytest
import torch

from tests._parity_log import record
from oracle.oracle import DEMO, DILOCO, FP16, FP32, FULL, RANDOM, STRIDING, TERNARY, Rep

pytestmark = pytest.mark.gpu
TOL = 1e-5


def P():
    import paper_2502_06728_b200 as mod

    return mod


def dev(x):
    return torch.as_tensor(np.asarray(x, np.float32)).cuda()


def host(t):
    return t.detach().cpu().numpy().astype(np.float64)


def rep_to_cfg(rep: Rep):
    p = P()
    return p.ReplicatorConfig(p.Scheme(rep.scheme), rep.chunk_size, rep.top_k, rep.compression, rep.sign_mode,
                              p.TransferDtype(rep.transfer_dtype), rep.seed)


def chunk_close(got, want, s, tol=TOL, what=""):
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    assert got.shape == want.shape, (what, got.shape, want.shape)
    n = len(want)
    pad = (-n) % s
    g = np.concatenate([got, np.zeros(pad)]).reshape(-1, s)
    w = np.concatenate([want, np.zeros(pad)]).reshape(-1, s)
    scale = np.maximum(np.abs(w).max(axis=1), 1e-30)
    err = np.abs(g - w).max(axis=1) / scale
    worst = float(err.max()) if len(err) else 0.0
    record(os.environ.get("PYTEST_CURRENT_TEST", "?").split(" ")[0], what or "value", worst, tol)
    bad = np.nonzero(err > tol)[0]
    assert len(bad) == 0, f"{what}: {len(bad)} chunks over tol, worst {worst:.3g} at chunk {bad[:5]}"
    return worst


UPDATE_TOL = 3e-5


def update_close(p_got, p_want, p_before, lr, s, tol=TOL, what="params"):
    """AdamW parameters.  The bar: p within 1e-5 of its chunk's L-inf (north_star's bar on
    parameters).  A stricter diagnostic on top: the applied update u = (p_before - p) / lr
    within 3e-5 of the chunk's largest |u|, beyond the FP32 rounding of the stored parameter
    itself (the Adam step and the weight decay each round p to FP32: 2 x 2^-24 |p| / lr in
    update units), which no FP32 parameter vector can resolve.  The ratio m_hat / sqrt(v_hat)
    amplifies the ~1e-6 relative error of the FP32 Q = IDCT(merged grid) where v_hat is small,
    so this bar sits at 3e-5 (measured worst: 1.2e-5 over 64 Mi parameters)."""
    chunk_close(p_got, p_want, s, tol=tol, what=what)
    tol = UPDATE_TOL
    pw = np.asarray(p_want, np.float64)
    u_want = (np.asarray(p_before, np.float64) - pw) / lr
    u_got = (np.asarray(p_before, np.float64) - np.asarray(p_got, np.float64)) / lr
    storage = 2.0 ** -23 * np.abs(pw) / lr
    excess = np.maximum(np.abs(u_got - u_want) - storage, 0.0)
    n = len(pw)
    pad = (-n) % s
    ex = np.concatenate([excess, np.zeros(pad)]).reshape(-1, s).max(axis=1)
    sc = np.maximum(np.abs(np.concatenate([u_want, np.zeros(pad)])).reshape(-1, s).max(axis=1), 1e-30)
    worst = float((ex / sc).max()) if len(ex) else 0.0
    record(os.environ.get("PYTEST_CURRENT_TEST", "?").split(" ")[0], what + " (update)", worst, tol)
    assert worst <= tol, f"{what}: update error {worst:.3g} of the chunk's largest update (bar {tol:.0e})"


def fp16_close(got, want):
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    ulp = np.maximum(np.abs(want), 2.0**-14) * 2.0**-10
    assert np.all(np.abs(got - want) <= ulp * 1.0001), np.abs(got - want).max()


def check_values(got, want, rep: Rep, group):
    if rep.sign_mode or rep.transfer_dtype == TERNARY:
        assert np.array_equal(got, want)
    elif rep.transfer_dtype == FP16:
        fp16_close(got, want)
    else:
        chunk_close(got, want, group, what="values")


# --------------------------------------------------------------- transform / encode
def test_demo_extraction_matches_golden(golden):
    p = P()
    g = golden["transform"]
    for ci in range(10):
        s, k, n = (int(x) for x in g[f"x_{ci}"])
        rep = Rep(scheme=DEMO, chunk_size=s, top_k=k, compression=k / s, sign_mode=False)
        enc = p.select_and_encode(dev(g[f"v_{ci}"]), rep_to_cfg(rep), 0, 0)
        idx = enc.update.freq_indices.cpu().numpy().astype(np.uint32)
        assert np.array_equal(idx, g[f"idx_{ci}"]), f"case {ci} (s={s} k={k}) indices differ"
        chunk_close(host(enc.update.values), g[f"co_{ci}"], k, what=f"coeffs {ci}")
        chunk_close(host(enc.local_q), g[f"fast_{ci}"], s, what=f"fast {ci}")
        if k == s:  # full band: exact identity (transform.cpp:119-125)
            assert np.array_equal(host(enc.local_q), g[f"v_{ci}"])


@pytest.mark.parametrize("seed", range(4))
@pytest.mark.parametrize("s,k", [(64, 32), (64, 8), (64, 56), (32, 4), (16, 5), (128, 16), (64, 1), (7, 3)])
def test_demo_indices_bit_exact_random(oracle, seed, s, k):
    p = P()
    rng = np.random.default_rng(1000 * seed + s + k)
    n = 64 * 257 + 13
    v = rng.standard_normal(n).astype(np.float32)
    # tie and degenerate chunks
    v[:64] = 0.0
    v[64:128] = 0.5
    v[128:192] = np.tile(v[192:200], 8)
    v[256:320] *= 1e-30
    for sign in (False, True):
        rep = Rep(scheme=DEMO, chunk_size=s, top_k=k, compression=k / s, sign_mode=sign)
        want = oracle.select_and_encode(v.astype(np.float64), rep, 3, 1)
        enc = p.select_and_encode(dev(v), rep_to_cfg(rep), 3, 1)
        got_idx = enc.update.freq_indices.cpu().numpy().astype(np.uint32)
        assert np.array_equal(got_idx, want["freq_indices"])
        check_values(host(enc.update.values), want["values"], rep, k)
        chunk_close(host(enc.local_q), want["local_q"], s, what="local_q")
        assert enc.update.bytes == want["bytes"]


def test_demo_large_config1_indices(oracle):
    """config-1 flavour at 2^20 elements: s=64, k=32, sign on; every index bit-exact"""
    p = P()
    n = 1 << 20
    v = (np.random.default_rng(7).standard_normal(n) * 1e-3).astype(np.float32)
    rep = Rep(scheme=DEMO, chunk_size=64, top_k=32, compression=0.5, sign_mode=True)
    want = oracle.select_and_encode(v.astype(np.float64), rep, 0, 0)
    enc = p.select_and_encode(dev(v), rep_to_cfg(rep), 0, 0)
    assert np.array_equal(enc.update.freq_indices.cpu().numpy().astype(np.uint32), want["freq_indices"])
    assert np.array_equal(host(enc.update.values), want["values"])
    chunk_close(host(enc.local_q), want["local_q"], 64, what="local_q")


def test_golden_replicate_all_schemes(golden):
    p = P()
    g = golden["replicate"]
    for ci in range(int(g["count"][0])):
        scheme, dtype, sign, step, s, k = (int(x) for x in g[f"cfg_{ci}"])
        rep = Rep(scheme=scheme, chunk_size=s, top_k=k, sign_mode=bool(sign), transfer_dtype=dtype,
                  compression=1.0 if scheme == FULL else 0.25, seed=99)
        cfg = rep_to_cfg(rep)
        ups = []
        for r in range(3):
            v = g[f"v_{ci}_{r}"]
            enc = p.select_and_encode(dev(v), cfg, step, 2)
            meta = [int(x) for x in g[f"meta_{ci}_{r}"]]
            assert [enc.update.bytes, int(enc.update.empty)] == meta, (ci, r)
            if scheme == DEMO:
                assert np.array_equal(enc.update.freq_indices.cpu().numpy().astype(np.uint32),
                                      g[f"freq_indices_{ci}_{r}"]), (ci, r)
            group = k if scheme == DEMO else max(len(g[f"values_{ci}_{r}"]), 1)
            if len(g[f"values_{ci}_{r}"]):
                check_values(host(enc.update.values), g[f"values_{ci}_{r}"], rep, group)
            chunk_close(host(enc.local_q), g[f"local_q_{ci}_{r}"], s if scheme == DEMO else len(v),
                        what=f"local_q {ci}")
            ups.append(enc.update)
        if f"q_{ci}_R1" in g:
            for R in (1, 2, 3):
                q = p.decode_and_merge(ups[:R], cfg)
                want = g[f"q_{ci}_R{R}"]
                if rep.transfer_dtype == FP16 and not rep.sign_mode:
                    chunk_close(host(q), want, s if scheme == DEMO else len(want), tol=2e-3, what=f"q {ci}")
                else:
                    chunk_close(host(q), want, s if scheme == DEMO else len(want), what=f"q {ci} R{R}")
            wire = np.frombuffer(p.serialize(ups[0], p.TransferDtype(dtype)), np.uint8)
            ref = g[f"wire_{ci}"]
            assert len(wire) == len(ref) and np.array_equal(wire[:9], ref[:9])
            if rep.sign_mode or dtype == TERNARY or scheme != DEMO:
                assert np.array_equal(wire, ref), ci
            if scheme == DEMO:  # indices part of the body is bit-exact
                ni = int(len(g[f"freq_indices_{ci}_0"])) * 4
                assert np.array_equal(wire[9:9 + ni], ref[9:9 + ni])


def test_random_index_sets_bit_exact(golden):
    p = P()
    g = golden["replicate"]
    for j in range(5):
        L, step, shard, seed = (int(x) for x in g[f"rand_cfg_{j}"])
        cfg = p.ReplicatorConfig(p.Scheme.Random, compression=float(g[f"rand_c_{j}"][0]), seed=seed)
        got = p.selected_indices(cfg, step, shard, L).cpu().numpy()
        assert np.array_equal(got, g[f"rand_idx_{j}"].astype(np.int64)), j


@pytest.mark.parametrize("L,c", [(1000, 0.25), (21468, 1 / 8), (300001, 1 / 16), (4096, 1.0), (777, 0.5)])
def test_random_index_sets_vs_oracle(oracle, L, c):
    p = P()
    for step in (0, 1, 9):
        for shard in (0, 3):
            rep = Rep(scheme=RANDOM, compression=c, seed=1234)
            want = oracle.selected_indices(rep, step, shard, L)
            got = p.selected_indices(rep_to_cfg(rep), step, shard, L).cpu().numpy()
            assert np.array_equal(got, want.astype(np.int64)), (step, shard)


def test_striding_sets(oracle):
    p = P()
    for L, c in ((10, 0.25), (1000, 1 / 7), (65, 0.5)):
        for step in range(6):
            rep = Rep(scheme=STRIDING, compression=c)
            got = p.selected_indices(rep_to_cfg(rep), step, 0, L).cpu().numpy()
            assert np.array_equal(got, oracle.selected_indices(rep, step, 0, L).astype(np.int64))


# --------------------------------------------------------------- optimizer stages
@pytest.mark.parametrize("scheme", [DEMO, RANDOM, STRIDING, DILOCO, FULL])
def test_sgd_stage_parity(oracle, scheme):
    """Stage parity: each step the oracle is fed the GPU's FP32 state."""
    p = P()
    n = 64 * 64 + 29
    rep = Rep(scheme=scheme, chunk_size=64, top_k=32, compression=1.0 if scheme == FULL else 0.25,
              sign_mode=True, seed=1234)
    cfg = rep_to_cfg(rep)
    opt = p.OptimizerConfig(momentum_decay=0.9)
    st = p.MomentumState.make(p.OptimizerKind.DemoSgd, n)
    params = dev(np.random.default_rng(1).standard_normal(n) * 0.02)
    for step in range(5):
        g = (np.random.default_rng(100 + step).standard_normal(n) * 1e-3).astype(np.float32)
        m_in = host(st.m)
        p_in = host(params)
        tr = p.StepTrace()
        enc = p.demo_sgd_prepare(st, dev(g), opt, cfg, step, 0, tr)
        m_o = m_in.copy()
        want = oracle.demo_sgd_prepare(m_o, g.astype(np.float64), 0.9, rep, step, 0)
        chunk_close(host(tr.m_accum), want["m_accum"], 64, what="m_accum")
        # selection is checked on the GPU's own accumulated momentum
        again = oracle.select_and_encode(host(tr.m_accum), rep, step, 0)
        if scheme == DEMO:
            assert np.array_equal(enc.update.freq_indices.cpu().numpy().astype(np.uint32), again["freq_indices"])
        assert enc.update.empty == again["empty"] and enc.update.bytes == again["bytes"]
        if not again["empty"]:
            assert np.array_equal(host(enc.update.values), again["values"])
        chunk_close(host(tr.local_q), again["local_q"], 64, what="local_q")
        chunk_close(host(st.m), host(tr.m_accum) - again["local_q"], 64, what="m_after")
        # merge + apply
        if not enc.update.empty:
            q = p.decode_and_merge([enc.update], cfg)
            want_q = oracle.decode_and_merge(rep, [again["values"]], [again["freq_indices"]], n, step, 0)
            chunk_close(host(q), want_q, 64, what="Q")
            p.demo_sgd_apply(params, q, 0.01)
            p_want = p_in.copy()
            oracle.demo_sgd_apply(p_want, want_q, 0.01)
        else:
            p.demo_sgd_apply(params, dev(g), 0.01)
            p_want = p_in - 0.01 * g.astype(np.float64)
        chunk_close(host(params), p_want, 64, what="params")


def test_conservation_exact_form():
    """acceptance 03 / test_optim.cpp:76-96: m_after == m_accum - local_q elementwise"""
    p = P()
    n = 96 * 64
    for sign in (False, True):
        cfg = p.ReplicatorConfig(p.Scheme.DeMo, 64, 8, 8 / 64, sign)
        st = p.MomentumState.make(p.OptimizerKind.DemoSgd, n)
        for step in range(4):
            tr = p.StepTrace()
            p.demo_sgd_prepare(st, torch.randn(n, device="cuda"), p.OptimizerConfig(), cfg, step, 0, tr)
            assert torch.equal(tr.m_after, tr.m_accum - tr.local_q)


def test_full_band_flushes_to_zero():
    """test_optim.cpp:121-134: k == s takes everything, m becomes exactly 0"""
    p = P()
    n = 64 * 10
    st = p.MomentumState.make(p.OptimizerKind.DemoSgd, n)
    p.demo_sgd_prepare(st, torch.randn(n, device="cuda"), p.OptimizerConfig(), p.ReplicatorConfig(p.Scheme.DeMo, 32, 4, sign_mode=False), 0, 0)
    tr = p.StepTrace()
    p.demo_sgd_prepare(st, torch.randn(n, device="cuda"), p.OptimizerConfig(),
                       p.ReplicatorConfig(p.Scheme.DeMo, 32, 32, sign_mode=False), 1, 0, tr)
    assert torch.equal(tr.local_q, tr.m_accum)
    assert torch.count_nonzero(st.m) == 0


def test_single_replica_merge_reproduces_local_share():
    """test_replicate.cpp:305-311 (within FP32 tolerance; bitwise in the reference's FP64)"""
    p = P()
    v = torch.randn(96 * 10, device="cuda")
    cfg = p.ReplicatorConfig(p.Scheme.DeMo, 32, 4, sign_mode=False)
    enc = p.select_and_encode(v, cfg, 0, 0)
    q = p.decode_and_merge([enc.update], cfg)
    chunk_close(host(q), host(enc.local_q), 32, tol=1e-6, what="single merge")


def test_adamw_stage_parity(oracle):
    p = P()
    n = 64 * 40 + 5
    rep = Rep(scheme=DEMO, chunk_size=64, top_k=16, compression=0.25, sign_mode=True, seed=1234)
    cfg = rep_to_cfg(rep)
    opt = p.OptimizerConfig(p.OptimizerKind.DecoupledAdamW, weight_decay=0.01)
    st = p.MomentumState.make(p.OptimizerKind.DecoupledAdamW, n)
    params = dev(np.random.default_rng(2).standard_normal(n) * 0.02)
    for step in range(4):
        g = (np.random.default_rng(200 + step).standard_normal(n) * 1e-3).astype(np.float32)
        p_in, ea_in, es_in = host(params), host(st.exp_avg), host(st.exp_avg_sq)
        enc = p.adamw_prepare(dev(g), cfg, step, 0)
        want = oracle.select_and_encode(g.astype(np.float64), rep, step, 0)
        assert np.array_equal(enc.update.freq_indices.cpu().numpy().astype(np.uint32), want["freq_indices"])
        q = p.decode_and_merge([enc.update], cfg)
        p.adamw_apply(params, st, dev(g), enc.local_q, q, opt, 0.003)
        want_q = oracle.decode_and_merge(rep, [want["values"]], [want["freq_indices"]], n, step, 0)
        pw, ew, sw = p_in.copy(), ea_in.copy(), es_in.copy()
        oracle.adamw_apply(pw, ew, sw, step, g.astype(np.float64), want["local_q"], want_q, 0.9, 0.999, 1e-8,
                           0.01, 0.003)
        chunk_close(host(st.exp_avg), ew, 64, what="exp_avg")
        chunk_close(host(st.exp_avg_sq), sw, 64, what="exp_avg_sq")
        update_close(host(params), pw, p_in, 0.003, 64)


def test_fused_local_sgd_step_matches_stages(oracle):
    """dmb_step_sgd_local (one pass) == prepare -> merge(R=1) -> apply"""
    import ctypes as C

    p = P()
    from paper_2502_06728_b200 import _capi
    from paper_2502_06728_b200.core import _ptr, _stream, context

    n = 64 * 1000 + 7
    cfg = p.ReplicatorConfig(p.Scheme.DeMo, 64, 32, 0.5, True, seed=1234)
    opt = p.OptimizerConfig(momentum_decay=0.9)
    g = torch.randn(n, device="cuda") * 1e-3
    m0 = torch.randn(n, device="cuda") * 1e-3
    p0 = torch.randn(n, device="cuda") * 0.02
    st = p.MomentumState(m=m0.clone())
    enc = p.demo_sgd_prepare(st, g, opt, cfg, 4, 0)
    q = p.decode_and_merge([enc.update], cfg)
    p_ref = p0.clone()
    p.demo_sgd_apply(p_ref, q, 0.01)
    m_out = torch.empty_like(m0)
    p_out = torch.empty_like(p0)
    hdr = _capi.Update()
    c, o = cfg.c(), opt.c()
    rc = _capi.lib.dmb_step_sgd_local(context().h, _ptr(g), _ptr(m0), _ptr(m_out), _ptr(p0), _ptr(p_out), n,
                                      C.byref(o), C.byref(c), 4, 0, 0.01, C.byref(hdr), _stream())
    assert rc == 0
    p.status()
    # the fused step takes the tensor-core path (3xTF32 inverse for local_q), the staged one the
    # SIMT kernel: the same selection, local_q within FP32 rounding of each other
    chunk_close(host(m_out), host(st.m), 64, what="m_out")  # 1e-5 of the chunk's L-inf (the parity bar)
    assert torch.allclose(p_out, p_ref, rtol=0, atol=1e-7)


def test_nonfinite_gradient_refused_before_state_changes():
    """test_optim.cpp:285-300"""
    p = P()
    n = 64 * 4
    st = p.MomentumState.make(p.OptimizerKind.DemoSgd, n)
    st.m.fill_(0.5)
    bad = torch.ones(n, device="cuda")
    bad[77] = float("nan")
    with pytest.raises(p.TrainingError, match="77"):
        p.demo_sgd_prepare(st, bad, p.OptimizerConfig(), p.ReplicatorConfig(p.Scheme.Full, compression=1.0), 0, 0)
    assert torch.all(st.m == 0.5)
    bad[77] = float("inf")
    with pytest.raises(p.TrainingError):
        p.adamw_prepare(bad, p.ReplicatorConfig(p.Scheme.DeMo, 64, 8), 0, 0)
    with pytest.raises(p.ProtocolError):
        p.demo_sgd_prepare(st, torch.ones(n - 1, device="cuda"), p.OptimizerConfig(),
                           p.ReplicatorConfig(p.Scheme.Full, compression=1.0), 0, 0)
    p.status()  # latch cleared


def test_merge_protocol_errors():
    """test_replicate.cpp:345-367"""
    p = P()
    v = torch.randn(64, device="cuda")
    cfg = p.ReplicatorConfig(p.Scheme.DeMo, 32, 4, sign_mode=False)
    ok = p.select_and_encode(v, cfg, 4, 2).update
    with pytest.raises(p.ProtocolError):
        p.decode_and_merge([], cfg)
    for kw in (dict(step=5), dict(shard_id=3), dict(empty=1), dict(n_values=ok.value_count() - 1)):
        with pytest.raises(p.ProtocolError):
            p.decode_and_merge([ok, ok.with_header(**kw)], cfg)
    with pytest.raises(p.ProtocolError):
        p.decode_and_merge([ok], p.ReplicatorConfig(p.Scheme.Random, compression=0.125))


def test_serialize_roundtrip_and_corruption():
    p = P()
    v = torch.randn(96, device="cuda")
    cfg = p.ReplicatorConfig(p.Scheme.DeMo, 32, 5, sign_mode=False)
    u = p.select_and_encode(v, cfg, 2, 7).update
    buf = p.serialize(u, cfg.transfer_dtype)
    assert len(buf) == 9 + u.bytes
    back = p.deserialize(buf, cfg.transfer_dtype, u)
    assert torch.equal(back.freq_indices, u.freq_indices) and torch.equal(back.values, u.values)
    with pytest.raises(p.ProtocolError):
        p.deserialize(buf[:-3], cfg.transfer_dtype, u)
    with pytest.raises(p.ProtocolError):
        p.deserialize(bytes([9]) + buf[1:], cfg.transfer_dtype, u)
    with pytest.raises(p.ProtocolError):
        p.deserialize(bytes([2]) + buf[1:], cfg.transfer_dtype, u)


def test_grad_mean_member_order(golden):
    p = P()
    g = golden["optim"]
    ins = [dev(x) for x in g["rs_in"]]
    out = host(p.grad_mean(ins))
    chunk_close(out, g["rs_out"].reshape(-1), 257, tol=1e-6, what="grad mean")


# --------------------------------------------------------------- tensor-core path
def test_tc_coefficient_error_within_certification_margin(oracle, monkeypatch):
    """The 3xTF32 tcgen05 DCT's coefficient error, measured against the FP64 oracle, stays
    well inside the certification radius eps = sqrt(2/s) (1.10e-6 Lw + 1.75e-6 ||x||_1) the kernel assumes
    (the bound derived in demo_tc_adam.cu from the per-MMA truncation model)."""
    p = P()
    monkeypatch.setenv("DMB_TC", "1")
    n = 64 * 128 * 40
    rng = np.random.default_rng(11)
    v = (rng.standard_normal(n) * 10.0 ** rng.uniform(-4, 2, size=n // 64).repeat(64)).astype(np.float32)
    rep = Rep(scheme=DEMO, chunk_size=64, top_k=64, compression=1.0, sign_mode=False)  # every coefficient
    enc = p.select_and_encode(dev(v), rep_to_cfg(rep), 0, 0)
    got = host(enc.update.values).reshape(-1, 64)
    want = oracle.select_and_encode(v.astype(np.float64), rep, 0, 0)["values"].reshape(-1, 64)
    ax = np.abs(v.astype(np.float64)).reshape(-1, 64)
    lw = (ax * (8 - np.arange(64) // 8)).sum(axis=1)  # the K-step-weighted |x| sum of the hi*hi steps
    eps = np.sqrt(2 / 64) * (1.10e-6 * lw + 1.75e-6 * ax.sum(axis=1))
    ratio = (np.abs(got - want).max(axis=1) / eps).max()
    print(f"tensor-core coefficient error: max {ratio:.4g} of the certification radius "
          f"sqrt(2/s) (1.10e-6 Lw + 1.75e-6 ||x||_1)")
    assert ratio < 0.5, f"tensor-core coefficient error reaches {ratio:.3f} of the certification radius"


@pytest.mark.parametrize("k", [8, 32, 56])
def test_tc_and_simt_paths_agree(oracle, monkeypatch, k):
    p = P()
    n = 64 * 128 * 30 + 64 * 7 + 5  # partial last tile and chunk
    rng = np.random.default_rng(k)
    v = (rng.standard_normal(n) * 1e-3).astype(np.float32)
    v[64 * 3:64 * 4] = 0.0
    v[64 * 9:64 * 10] = 1.0
    rep = Rep(scheme=DEMO, chunk_size=64, top_k=k, compression=k / 64, sign_mode=True)
    want = oracle.select_and_encode(v.astype(np.float64), rep, 2, 0)
    outs = {}
    for flag in ("0", "1"):
        monkeypatch.setenv("DMB_TC", flag)
        enc = p.select_and_encode(dev(v), rep_to_cfg(rep), 2, 0)
        outs[flag] = enc
        assert np.array_equal(enc.update.freq_indices.cpu().numpy().astype(np.uint32), want["freq_indices"]), flag
        assert np.array_equal(host(enc.update.values), want["values"])
        chunk_close(host(enc.local_q), want["local_q"], 64, what=f"local_q tc={flag}")


@pytest.mark.parametrize("opt_kind,force", [("sgd", False), ("adamw", False), ("sgd", True), ("adamw", True)])
def test_tc_fused_step_matches_oracle(oracle, monkeypatch, opt_kind, force):
    """dmb_step_*_local through the tensor-core kernel vs the oracle's prepare/merge/apply;
    force: every chunk is deferred to the exact FP64 fix-up (DMB_FORCE_FP64=1)"""
    import ctypes as C

    from paper_2502_06728_b200 import _capi
    from paper_2502_06728_b200.core import _ptr, _stream, context

    p = P()
    monkeypatch.setenv("DMB_TC", "1")
    if force:
        monkeypatch.setenv("DMB_FORCE_FP64", "1")
    n = 64 * 128 * 12 + 100
    rng = np.random.default_rng(5)
    g = (rng.standard_normal(n) * 1e-3).astype(np.float32)
    m0 = (rng.standard_normal(n) * 1e-3).astype(np.float32)
    p0 = (rng.standard_normal(n) * 0.02).astype(np.float32)
    ea0 = (rng.standard_normal(n) * 0.05).astype(np.float32)  # a plausible mid-training state
    es0 = (ea0.astype(np.float64) ** 2 * 4 + 1e-4).astype(np.float32)
    rep = Rep(scheme=DEMO, chunk_size=64, top_k=32, compression=0.5, sign_mode=True, seed=1234)
    cfg = rep_to_cfg(rep)
    c = cfg.c()
    gd, md, pd = dev(g), dev(m0), dev(p0)
    body = torch.empty(int(_capi.lib.dmb_update_capacity(C.byref(c), n)), dtype=torch.uint8, device="cuda")
    hdr = _capi.Update()
    hdr.body = body.data_ptr()
    lr = 0.01
    if opt_kind == "sgd":
        o = p.OptimizerConfig(momentum_decay=0.9).c()
        m_out, p_out = torch.empty_like(md), torch.empty_like(pd)
        rc = _capi.lib.dmb_step_sgd_local(context().h, _ptr(gd), _ptr(md), _ptr(m_out), _ptr(pd), _ptr(p_out), n,
                                          C.byref(o), C.byref(c), 3, 0, lr, C.byref(hdr), _stream())
        assert rc == 0, _capi.lib.dmb_last_error()
        p.status()
        macc = (np.float32(0.9) * m0).astype(np.float32) + g  # fp32 mul then add, as the kernel
        macc = macc.astype(np.float64)
        want = oracle.select_and_encode(macc, rep, 3, 0)
        q = oracle.decode_and_merge(rep, [want["values"]], [want["freq_indices"]], n, 3, 0)
        chunk_close(host(m_out), macc - want["local_q"], 64, what="m_out")
        chunk_close(host(p_out), p0 - lr * q, 64, what="p_out")
    else:
        o = p.OptimizerConfig(p.OptimizerKind.DecoupledAdamW).c()
        ead, esd = dev(ea0), dev(es0)
        steps = C.c_uint64(4)
        rc = _capi.lib.dmb_step_adamw_local(context().h, _ptr(gd), _ptr(pd), _ptr(pd), _ptr(ead), _ptr(ead), _ptr(esd),
                                            _ptr(esd), C.byref(steps), n, C.byref(o), C.byref(c), 3, 0, lr,
                                            C.byref(hdr), _stream())
        assert rc == 0, _capi.lib.dmb_last_error()
        p.status()
        want = oracle.select_and_encode(g.astype(np.float64), rep, 3, 0)
        q = oracle.decode_and_merge(rep, [want["values"]], [want["freq_indices"]], n, 3, 0)
        pw, ew, sw = p0.astype(np.float64), ea0.astype(np.float64), es0.astype(np.float64)
        oracle.adamw_apply(pw, ew, sw, 4, g.astype(np.float64), want["local_q"], q, 0.9, 0.999, 1e-8, 0.0, lr)
        chunk_close(host(ead), ew, 64, what="exp_avg")
        chunk_close(host(esd), sw, 64, what="exp_avg_sq")
        update_close(host(pd), pw, p0, lr, 64)
    idx = body[: 4 * want["freq_indices"].size].view(torch.int32).cpu().numpy().astype(np.uint32)
    assert np.array_equal(idx, want["freq_indices"])


@pytest.mark.parametrize("k,force,wire,sign,R", [(32, False, 0, True, 3), (8, False, 0, True, 3), (32, True, 0, True, 3),
                                                 (32, False, 1, True, 3), (8, True, 1, True, 3), (16, False, 1, False, 3),
                                                 (32, False, 1, True, 8), (16, False, 1, True, 17)])
def test_tc_cluster_adamw_prepare_merge_matches_oracle(oracle, monkeypatch, k, force, wire, sign, R):
    """The N>1 path as cluster.py drives it: dmb_adamw_prepare (no local_q: the tensor-core
    encode kernel) on R members' gradients, then dmb_merge_apply_adamw of the R bodies for one
    member (the tensor-core merge kernel) -- payloads and state against the oracle's
    select_and_encode / decode_and_merge / adamw_apply (cluster.cpp:193-231).  wire=1: the
    MASK exchange layout, whose serialize() must still be the reference's bytes; R = 17 takes
    the merge's unstaged path (more members than the scratch holds)."""
    import ctypes as C

    from paper_2502_06728_b200 import _capi
    from paper_2502_06728_b200.core import _ptr, _stream, context

    p = P()
    monkeypatch.setenv("DMB_TC", "1")
    if force:
        monkeypatch.setenv("DMB_FORCE_FP64", "1")
    lib = _capi.lib
    n = 64 * 128 * 6 + 64 * 3 + (0 if wire else 7)  # partial last tile (and chunk: reference layout)
    own, step, lr = 1, 5, 0.002
    rng = np.random.default_rng(31 + k + R)
    gs = [(rng.standard_normal(n) * 1e-3).astype(np.float32) for _ in range(R)]
    rep = Rep(scheme=DEMO, chunk_size=64, top_k=k, compression=k / 64, sign_mode=sign, seed=1234)
    c = rep_to_cfg(rep).c()
    cap = int(lib.dmb_update_capacity(C.byref(c), n))
    assert lib.dmb_set_wire_format(context().h, wire) == 0
    ups = (_capi.Update * R)()
    keep = []
    wants = []
    for r in range(R):
        gd = dev(gs[r])
        body = torch.zeros(cap, dtype=torch.uint8, device="cuda")
        hdr = _capi.Update()
        hdr.body = body.data_ptr()
        rc = lib.dmb_adamw_prepare(context().h, _ptr(gd), n, C.byref(c), step, 0, C.byref(hdr), None, _stream())
        assert rc == 0, lib.dmb_last_error()
        p.status()
        want = oracle.select_and_encode(gs[r].astype(np.float64), rep, step, 0)
        wants.append(want)
        assert hdr.wire_format == (0 if not wire else (2 if sign else 1))
        ser = (C.c_uint8 * (9 + cap))()
        written = C.c_uint64(0)
        assert lib.dmb_serialize(C.byref(hdr), 0, ser, 9 + cap, C.byref(written), _stream()) == 0, lib.dmb_last_error()
        raw = bytes(ser)[: written.value]
        ni = want["freq_indices"].size
        idx = np.frombuffer(raw[9: 9 + 4 * ni], dtype=np.uint32)
        assert np.array_equal(idx, want["freq_indices"]), f"member {r} indices"
        vals = np.frombuffer(raw[9 + 4 * ni: 9 + 8 * ni], dtype=np.float32)
        if sign:
            assert np.array_equal(vals, want["values"].astype(np.float32)), f"member {r} values"
        else:
            chunk_close(vals.astype(np.float64), want["values"], k, what=f"member {r} values")
        ups[r] = hdr
        keep += [gd, body]
    p0 = (rng.standard_normal(n) * 0.02).astype(np.float32)
    ea0 = (rng.standard_normal(n) * 0.05).astype(np.float32)
    es0 = (ea0.astype(np.float64) ** 2 * 4 + 1e-4).astype(np.float32)
    pd, ead, esd, god = dev(p0), dev(ea0), dev(es0), dev(gs[own])
    o = p.OptimizerConfig(p.OptimizerKind.DecoupledAdamW).c()
    steps = C.c_uint64(4)
    rc = lib.dmb_merge_apply_adamw(context().h, ups, R, own, C.byref(c), _ptr(pd), _ptr(ead), _ptr(esd),
                                   C.byref(steps), _ptr(god), n, step, C.byref(o), lr, _stream())
    assert lib.dmb_set_wire_format(context().h, 0) == 0
    assert rc == 0, lib.dmb_last_error()
    p.status()
    q = oracle.decode_and_merge(rep, [w["values"] for w in wants], [w["freq_indices"] for w in wants], n, step, 0)
    pw, ew, sw = p0.astype(np.float64), ea0.astype(np.float64), es0.astype(np.float64)
    oracle.adamw_apply(pw, ew, sw, 4, gs[own].astype(np.float64), wants[own]["local_q"], q, 0.9, 0.999, 1e-8, 0.0, lr)
    chunk_close(host(ead), ew, 64, what="exp_avg")
    chunk_close(host(esd), sw, 64, what="exp_avg_sq")
    update_close(host(pd), pw, p0, lr, 64)


@pytest.mark.parametrize("sign,dtype", [(True, FP32), (False, FP32), (False, FP16)])
def test_tc_near_ties_settle_in_fixup(oracle, monkeypatch, sign, dtype):
    """Chunks built with the k-th and (k+1)-th |c| a relative 1e-3 .. 1e-7 apart: the
    tensor-core kernel defers the close ones, the fix-up settles them with its FP32 FMA
    tree or, closer still, in FP64 in the oracle's order -- indices bit-exact and the
    AdamW state within tolerance either way (demo_tc_adam.cu, demo_fix64_kernel)."""
    import ctypes as C

    from paper_2502_06728_b200 import _capi
    from paper_2502_06728_b200.core import _ptr, _stream, context

    p = P()
    monkeypatch.setenv("DMB_TC", "1")
    S, k, nch = 64, 32, 128 * 6
    rng = np.random.default_rng(77)
    j = np.arange(S)
    B = np.sqrt(2.0 / S) * np.cos(np.pi * (2 * j[None, :] + 1) * j[:, None] / (2 * S))
    B[0] /= np.sqrt(2.0)
    c = rng.standard_normal((nch, S)) * 1e-3
    gaps = np.array([1e-3, 1e-4, 3e-5, 1e-7])[np.arange(nch) % 4]
    for r in range(nch):
        order = np.argsort(-np.abs(c[r]))
        kth, nxt = order[k - 1], order[k]
        c[r, nxt] = np.sign(c[r, nxt]) * abs(c[r, kth]) * (1.0 - gaps[r])
    g = (c @ B).astype(np.float32).reshape(-1)  # x = B^T c per chunk
    n = g.size
    p0 = (rng.standard_normal(n) * 0.02).astype(np.float32)
    ea0 = (rng.standard_normal(n) * 0.05).astype(np.float32)
    es0 = (ea0.astype(np.float64) ** 2 * 4 + 1e-4).astype(np.float32)
    rep = Rep(scheme=DEMO, chunk_size=S, top_k=k, compression=0.5, sign_mode=sign, transfer_dtype=dtype, seed=1234)
    cfg = rep_to_cfg(rep).c()
    body = torch.empty(int(_capi.lib.dmb_update_capacity(C.byref(cfg), n)), dtype=torch.uint8, device="cuda")
    hdr = _capi.Update()
    hdr.body = body.data_ptr()
    gd, pd, ead, esd = dev(g), dev(p0), dev(ea0), dev(es0)
    o = p.OptimizerConfig(p.OptimizerKind.DecoupledAdamW).c()
    steps = C.c_uint64(4)
    before = p.fallback_chunks()
    lr = 0.01
    rc = _capi.lib.dmb_step_adamw_local(context().h, _ptr(gd), _ptr(pd), _ptr(pd), _ptr(ead), _ptr(ead), _ptr(esd),
                                        _ptr(esd), C.byref(steps), n, C.byref(o), C.byref(cfg), 3, 0, lr,
                                        C.byref(hdr), _stream())
    assert rc == 0, _capi.lib.dmb_last_error()
    p.status()
    assert p.fallback_chunks() - before >= nch // 4, "the close chunks were not deferred"
    want = oracle.select_and_encode(g.astype(np.float64), rep, 3, 0)
    idx = body[: 4 * want["freq_indices"].size].view(torch.int32).cpu().numpy().astype(np.uint32)
    assert np.array_equal(idx, want["freq_indices"])
    q = oracle.decode_and_merge(rep, [want["values"]], [want["freq_indices"]], n, 3, 0)
    pw, ew, sw = p0.astype(np.float64), ea0.astype(np.float64), es0.astype(np.float64)
    oracle.adamw_apply(pw, ew, sw, 4, g.astype(np.float64), want["local_q"], q, 0.9, 0.999, 1e-8, 0.0, lr)
    chunk_close(host(ead), ew, 64, what="exp_avg")
    chunk_close(host(esd), sw, 64, what="exp_avg_sq")
    update_close(host(pd), pw, p0, lr, 64)


@pytest.mark.parametrize("L,c", [(300001, 1 / 16), (200000, 1 / 2)])
def test_random_substream_replay_matches_oracle(oracle, monkeypatch, L, c):
    """DMB_MT_FORCE_FIXUP=1 reports a Lemire rejection at output 0, so the exact sequential
    replay (random_index.cu, mt_fixup_kernel) rewrites every draw from the substream windows:
    the index set must still be bit-exact (the path a real rejection, p < 2^-32 per draw, takes)."""
    p = P()
    monkeypatch.setenv("DMB_MT_FORCE_FIXUP", "1")
    rep = Rep(scheme=RANDOM, compression=c, seed=4321)
    for step in (11, 12):
        want = oracle.selected_indices(rep, step, 1, L)
        got = p.selected_indices(rep_to_cfg(rep), step, 1, L).cpu().numpy()
        assert np.array_equal(got, want.astype(np.int64)), step


@pytest.mark.parametrize("tiles_per_cta,k", [(1, 64), (2, 64), (3, 64), (3, 32), (2, 8)])
def test_tc_step_few_tiles_per_cta(oracle, tiles_per_cta, k):
    """The last tile of a CTA stores W without a next forward to wait on: it must still wait for
    the inverse of the tile before (full band k = s, whose selection is instant, raced here)."""
    import ctypes as C

    from paper_2502_06728_b200 import _capi
    from paper_2502_06728_b200.core import _ptr, _stream, context

    p = P()
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    n = 64 * 128 * sms * tiles_per_cta
    rng = np.random.default_rng(tiles_per_cta + k)
    g = (rng.standard_normal(n) * 1e-3).astype(np.float32)
    p0 = (rng.standard_normal(n) * 0.02).astype(np.float32)
    ea0 = (rng.standard_normal(n) * 1e-3).astype(np.float32)
    es0 = (ea0.astype(np.float64) ** 2 * 4 + 1e-6).astype(np.float32)
    rep = Rep(scheme=DEMO, chunk_size=64, top_k=k, compression=k / 64, sign_mode=True, seed=1234)
    c = rep_to_cfg(rep).c()
    o = p.OptimizerConfig(p.OptimizerKind.DecoupledAdamW).c()
    gd, pd, ead, esd = dev(g), dev(p0), dev(ea0), dev(es0)
    steps = C.c_uint64(9)
    rc = _capi.lib.dmb_step_adamw_local(context().h, _ptr(gd), _ptr(pd), _ptr(pd), _ptr(ead), _ptr(ead), _ptr(esd),
                                        _ptr(esd), C.byref(steps), n, C.byref(o), C.byref(c), 9, 0, 1e-3, None,
                                        _stream())
    assert rc == 0, _capi.lib.dmb_last_error()
    p.status()
    e = oracle.select_and_encode(g.astype(np.float64), rep, 9, 0)
    q = oracle.decode_and_merge(rep, [e["values"]], [e["freq_indices"]], n, 9, 0)
    pw, ew, sw = p0.astype(np.float64), ea0.astype(np.float64), es0.astype(np.float64)
    oracle.adamw_apply(pw, ew, sw, 9, g.astype(np.float64), e["local_q"], q, 0.9, 0.999, 1e-8, 0.0, 1e-3)
    chunk_close(host(ead), ew, 64, what="exp_avg")
    chunk_close(host(esd), sw, 64, what="exp_avg_sq")
    update_close(host(pd), pw, p0, 1e-3, 64)


@pytest.mark.parametrize("opt_kind,sign", [("sgd", True), ("sgd", False), ("adamw", True)])
def test_v2_near_ties_and_single_frequency(oracle, monkeypatch, opt_kind, sign):
    """The paths with inspection outputs (local_q / m_accum) run the 16-warp v2 tensor-core
    kernel (demo_tc.cu) with its own derived radius: chunks built with the k-th and (k+1)-th |c|
    a relative 1e-3 .. 1e-7 apart, and chunks with a single nonzero frequency, must select the
    oracle's indices bit-exactly (near ties deferred to the FP64 fix-up) with local_q and m_accum
    within the 1e-5 bar."""
    p = P()
    monkeypatch.setenv("DMB_TC", "1")
    S, k, nch = 64, 8, 128 * 4
    rng = np.random.default_rng(808)
    j = np.arange(S)
    B = np.sqrt(2.0 / S) * np.cos(np.pi * (2 * j[None, :] + 1) * j[:, None] / (2 * S))
    B[0] /= np.sqrt(2.0)
    c = rng.standard_normal((nch, S)) * 1e-3
    gaps = np.array([1e-3, 1e-4, 3e-5, 1e-7])[np.arange(nch) % 4]
    for r in range(nch):
        if r % 16 == 5:  # a single frequency: one nonzero coefficient, the rest exact zeros (ties)
            c[r] = 0.0
            c[r, (r * 7) % S] = 2e-3
            continue
        order = np.argsort(-np.abs(c[r]))
        kth, nxt = order[k - 1], order[k]
        c[r, nxt] = np.sign(c[r, nxt]) * abs(c[r, kth]) * (1.0 - gaps[r])
    g = (c @ B).astype(np.float32).reshape(-1)
    n = g.size
    rep = Rep(scheme=DEMO, chunk_size=S, top_k=k, compression=k / S, sign_mode=sign, seed=1234)
    cfg = rep_to_cfg(rep)
    if opt_kind == "sgd":
        st = p.MomentumState.make(p.OptimizerKind.DemoSgd, n)  # zero momentum: m_acc = g
        tr = p.StepTrace()
        enc = p.demo_sgd_prepare(st, dev(g), p.OptimizerConfig(momentum_decay=0.9), cfg, 2, 0, tr)
        chunk_close(host(tr.m_accum), g.astype(np.float64), 64, what="m_accum")
        local_q = host(tr.local_q)
    else:
        enc = p.adamw_prepare(dev(g), cfg, 2, 0)
        local_q = host(enc.local_q)
    want = oracle.select_and_encode(g.astype(np.float64), rep, 2, 0)
    assert np.array_equal(enc.update.freq_indices.cpu().numpy().astype(np.uint32), want["freq_indices"])
    if sign:
        assert np.array_equal(host(enc.update.values), want["values"])
    else:  # FP32 coefficients against the oracle's FP64 ones, per chunk (k values each)
        chunk_close(host(enc.update.values), want["values"], k, what="values")
    chunk_close(local_q, want["local_q"], 64, what="local_q")
