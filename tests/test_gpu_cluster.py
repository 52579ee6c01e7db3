"""GPU parity of the N > 1 path: the tensor-core SGD encode / merge kernels through the C ABI,
and the bucketed HybridCluster pipeline driven with R x A in-process members on one GPU
(LocalHub: the members' bodies read in place, the shard-group mean by dmb_grad_mean),
against the reference's run_step_hybrid sequence (cluster.cpp:193-231) evaluated by the FP64
oracle on the same FP32 inputs: per member prepare, decode_and_merge of the R updates in
member order, apply.

Bars as in test_gpu_parity: indices bit-exact (through serialize), state within 1e-5 of its
chunk's L-inf; a refused step (non-finite gradient on one member) leaves every member's
parameters, momentum and moments as they were and raises TrainingError on every member.
"""
import ctypes as C
import os

import numpy as np
import pytest
import torch

from oracle.oracle import DEMO, DILOCO, FP16, FP32, RANDOM, STRIDING, Rep
from tests._parity_log import record

pytestmark = pytest.mark.gpu
TOL = 1e-5


def P():
    import paper_2502_06728_b200 as mod

    return mod


def chunk_rel(got, want, s=64):
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    pad = (-len(want)) % s
    g = np.concatenate([got, np.zeros(pad)]).reshape(-1, s)
    w = np.concatenate([want, np.zeros(pad)]).reshape(-1, s)
    return float((np.abs(g - w).max(axis=1) / np.maximum(np.abs(w).max(axis=1), 1e-30)).max()) if len(w) else 0.0


def check(what, err, tol=TOL):
    record(os.environ.get("PYTEST_CURRENT_TEST", "?").split(" ")[0], what, err, tol)
    assert err <= tol, f"{what}: {err:.3g} above {tol:.0e}"


def host(t):
    return t.detach().cpu().numpy().astype(np.float64)


def f32(x):
    return np.asarray(x, np.float64).astype(np.float32).astype(np.float64)


def macc32(m, g, beta):
    """the kernels' m_acc = beta m + g: FP32 multiply, then FP32 add (optim.cpp:27)"""
    return (np.float32(beta) * np.asarray(m, np.float32)).astype(np.float32) + np.asarray(g, np.float32)


def cfg_of(rep):
    p = P()
    return p.ReplicatorConfig(p.Scheme(rep.scheme), rep.chunk_size, rep.top_k, rep.compression, rep.sign_mode,
                              p.TransferDtype(rep.transfer_dtype), rep.seed)


# ------------------------------------------------------------- SGD kernels (C ABI)
@pytest.mark.parametrize("R,wire,sign,dtype", [(1, 1, True, FP32), (2, 1, True, FP32), (3, 1, True, FP32),
                                               (8, 1, True, FP32), (3, 0, True, FP32), (3, 1, False, FP32),
                                               (2, 1, False, FP16), (3, 0, False, FP32)])
def test_sgd_encode_merge_apply_matches_oracle(oracle, R, wire, sign, dtype):
    """dmb_demo_sgd_prepare (the tensor-core EncodeSgd kernel: no local_q output) on R members,
    then dmb_merge_apply_sgd of the R bodies (the tensor-core MergeSgd kernel) for one member:
    payload bytes, m_out and p against the oracle's demo_sgd_prepare / decode_and_merge /
    demo_sgd_apply (optim.cpp:18-49, replicate.cpp:239-314)."""
    from paper_2502_06728_b200 import _capi
    from paper_2502_06728_b200.core import _ptr, _stream, context

    p = P()
    lib = _capi.lib
    ctx = context().h
    n = 64 * 128 * 5 + 64 * 9 + (0 if wire else 21)  # partial tile (and partial chunk: reference layout)
    step, lr, beta, k = 4, 0.01, 0.9, 32
    rng = np.random.default_rng(7 + R + 10 * wire)
    rep = Rep(scheme=DEMO, chunk_size=64, top_k=k, compression=0.5, sign_mode=sign, transfer_dtype=dtype, seed=1234)
    c = cfg_of(rep).c()
    o = p.OptimizerConfig(momentum_decay=beta).c()
    cap = int(lib.dmb_update_capacity(C.byref(c), n))
    assert lib.dmb_set_wire_format(ctx, wire) == 0
    ups = (_capi.Update * R)()
    keep, wants = [], []
    try:
        for r in range(R):
            g = (rng.standard_normal(n) * 1e-3).astype(np.float32)
            m0 = (rng.standard_normal(n) * 1e-3).astype(np.float32)
            gd, md = torch.from_numpy(g).cuda(), torch.from_numpy(m0).cuda()
            m_out = torch.empty_like(md)
            body = torch.zeros(cap, dtype=torch.uint8, device="cuda")
            hdr = _capi.Update()
            hdr.body = body.data_ptr()
            rc = lib.dmb_demo_sgd_prepare(ctx, _ptr(gd), _ptr(md), _ptr(m_out), n, C.byref(o), C.byref(c), step, 0,
                                          C.byref(hdr), None, None, _stream())
            assert rc == 0, lib.dmb_last_error()
            p.status()
            want = oracle.select_and_encode(macc32(m0, g, beta).astype(np.float64), rep, step, 0)
            wants.append(want)
            exp_fmt = 0 if not wire or n % 64 else (2 if sign else 1)
            assert hdr.wire_format == exp_fmt
            ser = (C.c_uint8 * (9 + cap))()
            written = C.c_uint64(0)
            assert lib.dmb_serialize(C.byref(hdr), dtype, ser, 9 + cap, C.byref(written), _stream()) == 0
            raw = bytes(ser)[: written.value]
            ref = oracle.serialize(DEMO, want["freq_indices"], want["values"], dtype)
            ni = want["freq_indices"].size
            assert raw[: 9 + 4 * ni] == ref[: 9 + 4 * ni], f"member {r}: indices differ"
            if sign:
                assert raw == ref, f"member {r}: payload differs"
            elif dtype == FP16:  # the GPU rounds an FP32 coefficient, the oracle an FP64 one: 1 ulp
                got_v = np.frombuffer(raw[9 + 4 * ni: 9 + 6 * ni], np.float16).astype(np.float64)
                ulp = np.maximum(np.abs(want["values"]), 2.0 ** -14) * 2.0 ** -10
                assert np.all(np.abs(got_v - want["values"]) <= ulp * 1.0001), f"member {r}: fp16 values"
            check("m_out", chunk_rel(host(m_out), macc32(m0, g, beta) - want["local_q"]))
            ups[r] = hdr
            keep += [gd, md, m_out, body]
        p0 = (rng.standard_normal(n) * 0.02).astype(np.float32)
        pd = torch.from_numpy(p0).cuda()
        rc = lib.dmb_merge_apply_sgd(ctx, ups, R, C.byref(c), _ptr(pd), None, n, step, lr, _stream())
        assert rc == 0, lib.dmb_last_error()
        p.status()
    finally:
        lib.dmb_set_wire_format(ctx, 0)
    q = oracle.decode_and_merge(rep, [w["values"] for w in wants], [w["freq_indices"] for w in wants], n, step, 0)
    check("p", chunk_rel(host(pd), p0.astype(np.float64) - lr * q))


def test_sgd_merge_diloco_offbeat_applies_raw_gradient(oracle):
    """DiLoCo between beats: empty update, p -= lr g_shard (cluster.cpp:225)"""
    p = P()
    n = 10_000
    cfg = p.ReplicatorConfig(p.Scheme.DiLoCo, compression=0.25, seed=3)
    g = torch.randn(n, device="cuda") * 1e-3
    p0 = torch.randn(n, device="cuda") * 0.02
    pd = p0.clone()
    p.merge_apply_sgd([], cfg, pd, g, 1, 0.05)
    p.status()
    check("p (off-beat)", chunk_rel(host(pd), f32(host(p0) - 0.05 * host(g)), 10_000))


def test_sgd_merge_rejects_corrupt_mask_sign_body(oracle):
    """MASK_SIGN merges check every member's mask popcount and code words (replicate.cpp:284-293)"""
    from paper_2502_06728_b200 import _capi
    from paper_2502_06728_b200.core import _ptr, _stream, context

    p = P()
    lib = _capi.lib
    ctx = context().h
    n = 64 * 128 * 2
    rep = Rep(scheme=DEMO, chunk_size=64, top_k=16, compression=0.25, sign_mode=True, seed=1)
    c = cfg_of(rep).c()
    o = p.OptimizerConfig(momentum_decay=0.9).c()
    gd = torch.randn(n, device="cuda") * 1e-3
    md, mo = torch.zeros_like(gd), torch.zeros_like(gd)
    body = torch.zeros(int(lib.dmb_update_capacity(C.byref(c), n)), dtype=torch.uint8, device="cuda")
    hdr = _capi.Update()
    hdr.body = body.data_ptr()
    assert lib.dmb_set_wire_format(ctx, 1) == 0
    try:
        assert lib.dmb_demo_sgd_prepare(ctx, _ptr(gd), _ptr(md), _ptr(mo), n, C.byref(o), C.byref(c), 0, 0,
                                        C.byref(hdr), None, None, _stream()) == 0
    finally:
        lib.dmb_set_wire_format(ctx, 0)
    p.status()
    assert hdr.wire_format == 2
    for corrupt in ("mask", "code3"):
        bad = body.clone()
        if corrupt == "mask":
            bad[8 * 5] ^= 1  # chunk 5's mask loses / gains a frequency
        else:
            bad[8 * (n // 64) + 16 * 7] |= 3  # chunk 7, column 0: the invalid code 3
        h2 = _capi.Update.from_buffer_copy(hdr)
        h2.body = bad.data_ptr()
        ups = (_capi.Update * 2)(hdr, h2)
        pd = torch.zeros(n, device="cuda")
        assert lib.dmb_merge_apply_sgd(ctx, ups, 2, C.byref(c), _ptr(pd), None, n, 0, 0.1, _stream()) == 0
        with pytest.raises(p.ProtocolError):
            p.status()


# ------------------------------------------------------------- the cluster pipeline
def _oracle_hybrid_step(oracle, rep, opt_kind, members, shards, step, lr, beta=0.9):
    """run_step_hybrid (cluster.cpp:193-231) for one shard index on the oracle, fed each
    member's FP32 reduce-scattered shard gradient and pre-step state: returns per member
    (params, m or (exp_avg, exp_avg_sq))"""
    R = len(members)
    L = len(shards[0]["g"])
    encs = []
    for j in range(R):
        v = macc32(shards[j]["m"], shards[j]["g"], beta).astype(np.float64) if opt_kind == "sgd" else shards[j]["g"]
        encs.append(oracle.select_and_encode(v, rep, step, members[j]))
    empty = encs[0]["empty"]
    q = None if empty else oracle.decode_and_merge(rep, [e["values"] for e in encs],
                                                    [e["freq_indices"] for e in encs] if rep.scheme == DEMO else None,
                                                    L, step, members[0])
    out = []
    for j in range(R):
        sh = shards[j]
        pw = sh["p"].copy()
        if opt_kind == "sgd":
            macc = macc32(sh["m"], sh["g"], beta).astype(np.float64)
            m_after = macc - encs[j]["local_q"]
            oracle.demo_sgd_apply(pw, sh["g"] if empty else q, lr)
            out.append((pw, m_after))
        else:
            ew, sw = sh["ea"].copy(), sh["es"].copy()
            oracle.adamw_apply(pw, ew, sw, sh["steps"], sh["g"], encs[j]["local_q"], q, 0.9, 0.999, 1e-8, 0.0, lr)
            out.append((pw, (ew, sw)))
    return out


CASES = [
    # layout (A x R), optimizer, scheme, wire, sign, dtype
    ((1, 3), "adamw", DEMO, "mask", True, FP32),
    ((1, 3), "sgd", DEMO, "mask", True, FP32),
    ((2, 2), "adamw", DEMO, "mask", True, FP32),
    ((2, 2), "sgd", DEMO, "reference", False, FP16),
    ((1, 2), "sgd", DEMO, "mask", False, FP32),
    ((2, 1), "adamw", DEMO, "mask", True, FP32),  # R = 1: the fused step, double buffered
    ((2, 1), "sgd", DEMO, "mask", True, FP32),
    ((1, 3), "sgd", RANDOM, "mask", False, FP32),
    ((1, 2), "adamw", STRIDING, "mask", False, FP16),
    ((1, 2), "sgd", DILOCO, "mask", False, FP32),
]


def _make_cluster(layout, opt_kind, scheme, wire, sign, dtype, param_count, p0):
    p = P()
    from paper_2502_06728_b200.cluster import HybridCluster, LocalExchange, LocalHub, Topology

    A, R = layout
    topo = Topology(nodes=R, accels_per_node=A)
    hub = LocalHub(topo)
    k = 32 if scheme == DEMO else 0
    rep = Rep(scheme=scheme, chunk_size=64, top_k=max(k, 1), compression=0.5 if scheme == DEMO else 0.25,
              sign_mode=sign, transfer_dtype=dtype, seed=1234)
    opt = p.OptimizerConfig(p.OptimizerKind.DemoSgd if opt_kind == "sgd" else p.OptimizerKind.DecoupledAdamW,
                            momentum_decay=0.9)
    members = [HybridCluster(topo, param_count, opt, cfg_of(rep), p0, r, buckets=3, wire=wire,
                             exchange=LocalExchange(hub, r)) for r in range(topo.world_size)]
    return topo, hub, rep, members


@pytest.mark.parametrize("layout,opt_kind,scheme,wire,sign,dtype", CASES)
def test_hybrid_cluster_pipeline_matches_oracle(oracle, layout, opt_kind, scheme, wire, sign, dtype):
    A, R = layout
    param_count = 64 * 128 * 5 + 64 * 3 + 17  # shards with a partial last tile and chunk
    rng = np.random.default_rng(hash((layout, opt_kind, scheme, wire)) & 0xFFFF)
    p0 = torch.from_numpy((rng.standard_normal(param_count) * 0.02).astype(np.float32)).cuda()
    topo, hub, rep, members = _make_cluster(layout, opt_kind, scheme, wire, sign, dtype, param_count, p0)
    padded = members[0].spec.extent * A
    lr = 0.01
    if opt_kind == "adamw":  # a mid-training state: Adam's first steps from zero are ill-conditioned
        for m in members:
            ea = rng.standard_normal(m.spec.real_len) * 1e-3
            m.exp_avg.copy_(torch.from_numpy(ea.astype(np.float32)))
            m.exp_avg_sq.copy_(torch.from_numpy((4 * ea * ea + 1e-6).astype(np.float32)))
            m.steps = 9
    for step in range(2):
        grads = [torch.from_numpy((rng.standard_normal(padded) * 1e-3).astype(np.float32)).cuda()
                 for _ in range(topo.world_size)]
        before = []
        for r, m in enumerate(members):
            hub.grads[r] = grads[r]
            st = dict(p=host(m.params), steps=m.steps)
            if opt_kind == "sgd":
                st["m"] = host(m.m)
            else:
                st["ea"], st["es"] = host(m.exp_avg), host(m.exp_avg_sq)
            before.append(st)
        for m in members:
            m.begin(step, lr, grads[m.rank])
        hub.agree()
        for m in members:
            m.commit()
        for accel in range(A):  # one replica group per shard index
            ranks = [n * A + accel for n in range(R)]
            shards = []
            for r in ranks:
                L = members[r].spec.real_len
                sh = dict(before[r])
                # the reduce-scatter: member-order mean of the node's gradients, FP32 on the device
                node = r // A
                full = [host(grads[node * A + a]) for a in range(A)]
                sh["g"] = host(members[r].g_shard)
                want_g = np.mean([f[accel * members[r].spec.extent:][:L] for f in full], axis=0)
                check("reduce-scatter", chunk_rel(sh["g"], want_g), 1e-6)
                shards.append(sh)
            want = _oracle_hybrid_step(oracle, rep, opt_kind, [accel] * R, shards, step, lr)
            for j, r in enumerate(ranks):
                m = members[r]
                check(f"params step {step}", chunk_rel(host(m.params), want[j][0]))
                if opt_kind == "sgd":
                    check(f"momentum step {step}", chunk_rel(host(m.m), want[j][1]))
                else:
                    check(f"exp_avg step {step}", chunk_rel(host(m.exp_avg), want[j][1][0]))
                    check(f"exp_avg_sq step {step}", chunk_rel(host(m.exp_avg_sq), want[j][1][1]))
                    assert m.steps == before[r]["steps"] + 1
        tr = members[0].ledger[-1]
        if R > 1 and scheme == DEMO:
            assert tr.inter_bytes_reference >= tr.inter_bytes > 0


@pytest.mark.parametrize("opt_kind,layout", [("sgd", (1, 3)), ("adamw", (2, 2)), ("adamw", (2, 1))])
def test_hybrid_cluster_refuses_nonfinite_step_everywhere(opt_kind, layout):
    """A NaN in one member's gradient: every member's step is refused (TrainingError) and no
    state changes anywhere (optim.cpp:21, cluster.cpp:182), across the buckets; the next
    clean step then runs normally."""
    p = P()
    A, R = layout
    param_count = 64 * 128 * 6
    rng = np.random.default_rng(5)
    p0 = torch.from_numpy((rng.standard_normal(param_count) * 0.02).astype(np.float32)).cuda()
    topo, hub, rep, members = _make_cluster(layout, opt_kind, DEMO, "mask", True, FP32, param_count, p0)
    padded = members[0].spec.extent * A
    grads = [torch.randn(padded, device="cuda") * 1e-3 for _ in range(topo.world_size)]
    for r, m in enumerate(members):  # one clean step first: non-trivial state
        hub.grads[r] = grads[r]
    for r, m in enumerate(members):
        m.begin(0, 0.01, grads[r])
    hub.agree()
    for m in members:
        m.commit()
    snap = [[host(t) for t in ((m.params, m.m) if opt_kind == "sgd" else (m.params, m.exp_avg, m.exp_avg_sq))]
            for m in members]
    steps = [m.steps for m in members]
    bad = [g.clone() for g in grads]
    bad[topo.world_size - 1][padded - 100] = float("nan")  # last bucket of the last member
    for r, m in enumerate(members):
        hub.grads[r] = bad[r]
    for r, m in enumerate(members):
        m.begin(1, 0.01, bad[r])
    hub.agree()
    for m in members:
        with pytest.raises(p.TrainingError):
            m.commit()
    for m, sn, s0 in zip(members, snap, steps):
        now = [host(t) for t in ((m.params, m.m) if opt_kind == "sgd" else (m.params, m.exp_avg, m.exp_avg_sq))]
        for a, b in zip(now, sn):
            assert np.array_equal(a, b), "a refused step changed state"
        assert m.steps == s0
    for r, m in enumerate(members):  # the next clean step runs
        hub.grads[r] = grads[r]
    for r, m in enumerate(members):
        m.begin(2, 0.01, grads[r])
    hub.agree()
    for m in members:
        m.commit()
