"""Generate tests/golden/*.npz from the UNMODIFIED reference build.

TEST INFRASTRUCTURE ONLY.  Run here (where /root/reference exists):

    make -C oracle ref && python oracle/gen_golden.py

Every array in the fixtures is an output of oracle/_ref/libdemosim_ref.so (the
reference core compiled where it lies, plus the extern-"C" shim ref_shim.cpp) on
seeded inputs; tests/test_oracle_golden.py pins the C restatement to them and the
GPU parity tests reuse the inputs.  Inputs are FP32-representable so the same
vectors drive the FP32 device path.
"""
from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.oracle import (DEMO, DILOCO, FP16, FP32, FULL, RANDOM, STRIDING, TERNARY,  # noqa: E402
                           Rep, reference)

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")


def f32(v):
    return np.asarray(v, np.float64).astype(np.float32).astype(np.float64)


def main():
    ref = reference()
    if ref is None:
        raise SystemExit("oracle/_ref/libdemosim_ref.so missing: run `make -C oracle ref` first")
    os.makedirs(OUT, exist_ok=True)

    # --- rng: engine KAT and derived draws (rng.hpp:19-51) ---------------------
    ns = np.array([1, 2, 3, 10, 1000, 2**31 + 11, 2**40 + 3, 21468889, 55725888, 2**63 + 5], np.uint64)
    np.savez_compressed(
        os.path.join(OUT, "rng.npz"),
        mt_default=ref.mt64_stream(5489, 10000),
        mix=np.array([ref.mix_seed(1234), ref.mix_seed(1234, 7), ref.mix_seed(1234, 7, 3),
                      ref.mix_seed(99, 5, 2)], np.uint64),
        below_ns=ns, below=ref.rng_below(42, np.tile(ns, 20)),
        normal_11=ref.random_vector(11, 257), normal_1234=ref.random_vector(1234, 64),
    )

    # --- transform: basis, extraction incl. ties / pads / full band -----------
    tr = {}
    for s in (1, 2, 7, 8, 16, 32, 64, 128):
        tr[f"basis_{s}"] = ref.dct_basis(s)
    cases = [(64, 32, 4096 + 17), (64, 8, 3000), (64, 64, 640), (32, 4, 96), (32, 32, 70), (16, 5, 160),
             (8, 3, 8), (7, 2, 50), (128, 16, 1000), (64, 1, 200)]
    for ci, (s, k, n) in enumerate(cases):
        v = f32(ref.random_vector(5000 + ci, n))
        if ci == 0:
            v[64:128] = 0.0           # an all-zero chunk: every coefficient ties
            v[128:192] = 0.25         # a constant chunk: exact ties in the high band
            v[192:256] = v[0:64]      # a duplicated chunk
        idx, co, fast, res = ref.extract(v, s, k)
        tr[f"x_{ci}"] = np.array([s, k, n])
        tr[f"v_{ci}"], tr[f"idx_{ci}"], tr[f"co_{ci}"] = v, idx, co
        tr[f"fast_{ci}"], tr[f"res_{ci}"] = fast, res
    np.savez_compressed(os.path.join(OUT, "transform.npz"), **tr)

    # --- replicate: every scheme x dtype x sign, encode + R-way merge + bytes ---
    rp = {}
    n = 300
    ci = 0
    for scheme in (DEMO, RANDOM, STRIDING, DILOCO, FULL):
        for dtype in (FP32, FP16, TERNARY):
            for sign in (False, True):
                rep = Rep(scheme=scheme, chunk_size=64, top_k=8, sign_mode=sign, transfer_dtype=dtype,
                          compression=1.0 if scheme == FULL else 0.25, seed=99)
                for step in (0, 5):
                    vs, ids, encs = [], [], []
                    for r in range(3):
                        v = f32(ref.random_vector(7000 + 10 * ci + r, n))
                        e = ref.select_and_encode(v, rep, step, 2)
                        rp[f"v_{ci}_{r}"] = v.astype(np.float32)
                        for key in ("freq_indices", "values", "local_q"):
                            rp[f"{key}_{ci}_{r}"] = e[key]
                        rp[f"meta_{ci}_{r}"] = np.array([e["bytes"], int(e["empty"])], np.uint64)
                        vs.append(e["values"])
                        ids.append(e["freq_indices"])
                        encs.append(e)
                    rp[f"cfg_{ci}"] = np.array([scheme, dtype, int(sign), step, 64, 8], np.int64)
                    if not encs[0]["empty"]:
                        for R in (1, 2, 3):
                            rp[f"q_{ci}_R{R}"] = ref.decode_and_merge(rep, vs[:R], ids[:R], n, step, 2)
                        rp[f"wire_{ci}"] = np.frombuffer(
                            ref.serialize(scheme, ids[0], vs[0], dtype), np.uint8)
                    ci += 1
    rp["count"] = np.array([ci])
    # Random index sets at larger sizes (no literal vectors exist in the reference tests)
    for j, (L, c, step, shard) in enumerate([(1600, 1 / 16, 5, 2), (128, 1 / 16, 7, 1), (100003, 1 / 8, 3, 0),
                                             (65536, 1 / 2, 0, 3), (1 << 20, 1 / 32, 11, 1)]):
        rep = Rep(scheme=RANDOM, compression=c, seed=99 if j < 2 else 1234)
        rp[f"rand_cfg_{j}"] = np.array([L, step, shard, rep.seed], np.uint64)
        rp[f"rand_c_{j}"] = np.array([c])
        rp[f"rand_idx_{j}"] = ref.selected_indices(rep, step, shard, L)
    np.savez_compressed(os.path.join(OUT, "replicate.npz"), **rp)

    # --- optim trajectories: DeMo-SGD (config-1 flavour) and decoupled AdamW --
    op = {}
    L = 64 * 24 + 13
    rep = Rep(scheme=DEMO, chunk_size=64, top_k=32, compression=0.5, sign_mode=True, seed=1234)
    m = np.zeros(L)
    p = f32(0.02 * ref.random_vector(1, L))
    op["sgd_p0"] = p.copy()
    for step in range(4):
        g = f32(1e-3 * ref.random_vector(100 + step, L))
        e = ref.demo_sgd_prepare(m, g, 0.9, rep, step, 0)
        q = ref.decode_and_merge(rep, [e["values"]], [e["freq_indices"]], L, step, 0)
        ref.demo_sgd_apply(p, q, 0.01)
        op[f"sgd_g_{step}"] = g
        for key in ("freq_indices", "values", "local_q", "m_accum", "m_after"):
            op[f"sgd_{key}_{step}"] = e[key]
        op[f"sgd_q_{step}"], op[f"sgd_p_{step}"] = q, p.copy()
    rep_a = Rep(scheme=DEMO, chunk_size=64, top_k=16, compression=0.25, sign_mode=True, seed=1234)
    p = f32(0.02 * ref.random_vector(2, L))
    ea, es = np.zeros(L), np.zeros(L)
    steps = 0
    op["adam_p0"] = p.copy()
    for step in range(4):
        g = f32(1e-3 * ref.random_vector(200 + step, L))
        e = ref.select_and_encode(g, rep_a, step, 0)
        q = ref.decode_and_merge(rep_a, [e["values"]], [e["freq_indices"]], L, step, 0)
        steps = ref.adamw_apply(p, ea, es, steps, g, e["local_q"], q, 0.9, 0.999, 1e-8, 0.01, 0.003)
        op[f"adam_g_{step}"], op[f"adam_q_{step}"], op[f"adam_lq_{step}"] = g, q, e["local_q"]
        op[f"adam_idx_{step}"], op[f"adam_vals_{step}"] = e["freq_indices"], e["values"]
        op[f"adam_p_{step}"], op[f"adam_ea_{step}"], op[f"adam_es_{step}"] = p.copy(), ea.copy(), es.copy()
    gs = [f32(ref.random_vector(300 + a, 4 * 257)) for a in range(4)]
    op["rs_in"] = np.stack(gs).astype(np.float32)
    op["rs_out"] = ref.grad_reduce_scatter(gs)
    np.savez_compressed(os.path.join(OUT, "optim.npz"), **op)
    for f in sorted(os.listdir(OUT)):
        print(f, os.path.getsize(os.path.join(OUT, f)))


if __name__ == "__main__":
    main()
