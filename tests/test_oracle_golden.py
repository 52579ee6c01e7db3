"""Pin the C restatement (oracle/demo_oracle.c) before trusting it.

(1) literal known answers from the reference's own tests, (2) golden vectors
produced by the unmodified reference build (tests/golden/, oracle/gen_golden.py),
(3) when oracle/_ref exists (this container), a randomized differential run of
restatement vs reference.  All comparisons are bit-exact.
"""
import math

import numpy as np
import pytest

from oracle.oracle import (CONFIG, DEMO, DILOCO, FP16, FP32, FULL, PROTOCOL, RANDOM, STRIDING,
                           TERNARY, OracleError, Rep, reference)


def eq(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return a.shape == b.shape and np.array_equal(a.view(np.uint8) if a.dtype == b.dtype else a, b.view(
        np.uint8) if a.dtype == b.dtype else b)


# ---------------------------------------------------------------- known answers
def test_mt19937_64_known_answer(oracle):
    # [rand.predef]: 10000th output of a default-constructed mt19937_64 (SURVEY §7 KAT)
    assert int(oracle.mt64_stream(5489, 10000)[-1]) == 9981545732273789042


def test_wire_bytes_literals(oracle):
    # test_replicate.cpp:47-62
    assert oracle.wire_bytes(100, 0, FP32) == 400
    assert oracle.wire_bytes(100, 0, FP16) == 200
    assert oracle.wire_bytes(100, 0, TERNARY) == 25
    assert oracle.wire_bytes(3, 0, TERNARY) == 1
    assert oracle.wire_bytes(16, 16, FP32) == 128
    assert oracle.wire_bytes(0, 0, FP32) == 0
    assert oracle.wire_bytes(100, 100, FP32) == 800
    assert oracle.wire_bytes(1600, 0, FP32) == 6400


def test_period_literals(oracle):
    # test_replicate.cpp:64-74
    assert oracle.period(0.125) == 8
    assert oracle.period(1.0 / 3.0) == 3
    assert oracle.period(1.0) == 1
    assert oracle.period(2.0) == 1


def test_striding_literals(oracle):
    # test_replicate.cpp:139-158
    rep = Rep(scheme=STRIDING, compression=0.25, sign_mode=False, seed=99)
    assert list(oracle.selected_indices(rep, 0, 0, 10)) == [0, 4, 8]
    assert list(oracle.selected_indices(rep, 1, 0, 10)) == [1, 5, 9]
    assert list(oracle.selected_indices(rep, 2, 0, 10)) == [2, 6]
    assert list(oracle.selected_indices(rep, 3, 0, 10)) == [3, 7]
    assert list(oracle.selected_indices(rep, 5, 0, 10)) == [1, 5, 9]
    with pytest.raises(OracleError) as e:
        oracle.selected_indices(rep, 0, 0, 3)
    assert e.value.code == CONFIG


def test_constant_chunk_and_zero_ties(oracle):
    # test_transform.cpp:114-119: DCT of ones(4) has c0 == 2
    b = oracle.dct_basis(4)
    c = b @ np.ones(4)
    assert abs(c[0] - 2.0) <= 2.0 * 1e-14 and np.all(np.abs(c[1:]) < 1e-15)
    # test_transform.cpp:142-150: all-zero input selects {0,1,2}
    idx, co, fast, res = oracle.extract(np.zeros(8), 8, 3)
    assert list(idx) == [0, 1, 2]


def test_sign_transform_alphabet(oracle):
    # test_transform.cpp:214-223
    v = oracle.sign_transform([3.5, -0.25, 0.0, -0.0, 1e-300, -1e-300, math.inf, -math.inf, math.nan])
    assert list(v) == [1.0, -1.0, 0.0, 0.0, 1.0, -1.0, 1.0, -1.0, 0.0]
    assert not math.copysign(1.0, v[3]) < 0


def test_fp16_narrowing_literals(oracle):
    # test_replicate.cpp:180-192
    n = oracle.narrow_fp16
    assert n(0.0) == 0.0 and n(1.0) == 1.0 and n(65504.0) == 65504.0
    assert math.isinf(n(65520.0)) and math.isinf(n(1e6)) and n(-65520.0) == -math.inf
    assert n(2.0**-24) == 2.0**-24 and n(2.0**-25) == 0.0
    assert n(1.0 + 2.0**-11) == 1.0 and n(1.0 + 3 * 2.0**-11) == 1.0 + 2.0**-9
    assert math.isnan(n(math.nan))
    assert oracle.narrow_fp32(0.1) == float(np.float32(0.1)) and math.isinf(oracle.narrow_fp32(1e39))


def test_serialization_literals(oracle):
    # test_replicate.cpp:218-252
    buf = oracle.serialize(FULL, None, [1.0, -2.0], FP32)
    assert len(buf) == 9 + 8 and buf[0] == 5 and buf[1] == 2 and all(x == 0 for x in buf[2:9])
    assert list(buf[9:13]) == [0x00, 0x00, 0x80, 0x3F]
    assert oracle.serialize(FULL, None, [1.0, -1.0, 0.0, 1.0], TERNARY)[9] == 0x49


def test_acceptance_byte_ratios(oracle):
    # acceptance_test.cpp:353-399 (criterion 05): 800 / 400 / 6400 / 25 / 200 bytes
    v = oracle.random_vector(500, 1600)
    demo = Rep(scheme=DEMO, chunk_size=32, top_k=2, compression=1 / 16, sign_mode=True)
    rnd = Rep(scheme=RANDOM, compression=1 / 16, sign_mode=True, seed=3)
    full = Rep(scheme=FULL, compression=1.0, sign_mode=False)
    assert oracle.select_and_encode(v, demo, 0, 0)["bytes"] == 800
    assert oracle.select_and_encode(v, rnd, 0, 0)["bytes"] == 400
    assert oracle.select_and_encode(v, full, 0, 0)["bytes"] == 6400
    rnd.transfer_dtype = TERNARY
    assert oracle.select_and_encode(v, rnd, 0, 0)["bytes"] == 25
    rnd.transfer_dtype = FP16
    assert oracle.select_and_encode(v, rnd, 0, 0)["bytes"] == 200


def test_random_selection_properties(oracle):
    # test_replicate.cpp:107-137
    rep = Rep(scheme=RANDOM, compression=1 / 16, sign_mode=False, seed=99)
    a = oracle.selected_indices(rep, 5, 2, 1600)
    assert len(a) == 100 and np.all(np.diff(a.astype(np.int64)) > 0) and a[-1] < 1600
    assert not np.array_equal(oracle.selected_indices(rep, 6, 2, 1600), a)
    assert not np.array_equal(oracle.selected_indices(rep, 5, 3, 1600), a)
    with pytest.raises(OracleError):
        oracle.selected_indices(Rep(scheme=RANDOM, compression=1e-6, seed=99), 0, 0, 100)


def test_diloco_beat(oracle):
    # test_replicate.cpp:160-178
    rep = Rep(scheme=DILOCO, compression=0.25, sign_mode=False, seed=99)
    v = oracle.random_vector(14, 40)
    for step in range(9):
        e = oracle.select_and_encode(v, rep, step, 0)
        if step % 4 == 0:
            assert not e["empty"] and eq(e["values"], v) and eq(e["local_q"], v) and e["bytes"] == 160
        else:
            assert e["empty"] and len(e["values"]) == 0 and e["bytes"] == 0 and not e["local_q"].any()


def test_merge_length_mismatch_is_protocol_error(oracle):
    rep = Rep(scheme=DEMO, chunk_size=32, top_k=4, sign_mode=False)
    v = oracle.random_vector(21, 64)
    e = oracle.select_and_encode(v, rep, 4, 2)
    with pytest.raises(OracleError) as ex:
        oracle.decode_and_merge(rep, [e["values"][:-1]], [e["freq_indices"][:-1]], 64, 4, 2)
    assert ex.value.code == PROTOCOL


# ---------------------------------------------------------------- golden vectors
def test_golden_rng(oracle, golden):
    g = golden["rng"]
    assert eq(oracle.mt64_stream(5489, 10000), g["mt_default"])
    assert [oracle.mix_seed(1234), oracle.mix_seed(1234, 7), oracle.mix_seed(1234, 7, 3),
            oracle.mix_seed(99, 5, 2)] == [int(x) for x in g["mix"]]
    assert eq(oracle.rng_below(42, np.tile(g["below_ns"], 20)), g["below"])
    assert eq(oracle.random_vector(11, 257), g["normal_11"])
    assert eq(oracle.random_vector(1234, 64), g["normal_1234"])


def test_golden_transform(oracle, golden):
    g = golden["transform"]
    for s in (1, 2, 7, 8, 16, 32, 64, 128):
        assert eq(oracle.dct_basis(s), g[f"basis_{s}"]), s
    ci = 0
    while f"x_{ci}" in g:
        s, k, n = (int(x) for x in g[f"x_{ci}"])
        idx, co, fast, res = oracle.extract(g[f"v_{ci}"], s, k)
        assert eq(idx, g[f"idx_{ci}"]) and eq(co, g[f"co_{ci}"]), ci
        assert eq(fast, g[f"fast_{ci}"]) and eq(res, g[f"res_{ci}"]), ci
        ci += 1
    assert ci == 10


def _rep_from(cfg):
    scheme, dtype, sign, step, s, k = (int(x) for x in cfg)
    return Rep(scheme=scheme, chunk_size=s, top_k=k, sign_mode=bool(sign), transfer_dtype=dtype,
               compression=1.0 if scheme == FULL else 0.25, seed=99), step


def test_golden_replicate(oracle, golden):
    g = golden["replicate"]
    for ci in range(int(g["count"][0])):
        rep, step = _rep_from(g[f"cfg_{ci}"])
        vs, ids = [], []
        for r in range(3):
            e = oracle.select_and_encode(g[f"v_{ci}_{r}"].astype(np.float64), rep, step, 2)
            for key in ("freq_indices", "values", "local_q"):
                assert eq(e[key], g[f"{key}_{ci}_{r}"]), (ci, r, key)
            assert [e["bytes"], int(e["empty"])] == [int(x) for x in g[f"meta_{ci}_{r}"]]
            vs.append(e["values"])
            ids.append(e["freq_indices"])
        if f"q_{ci}_R1" in g:
            n = len(g[f"v_{ci}_0"])
            for R in (1, 2, 3):
                assert eq(oracle.decode_and_merge(rep, vs[:R], ids[:R], n, step, 2), g[f"q_{ci}_R{R}"])
            wire = np.frombuffer(oracle.serialize(rep.scheme, ids[0], vs[0], rep.transfer_dtype), np.uint8)
            assert eq(wire, g[f"wire_{ci}"]), ci


def test_golden_random_index_sets(oracle, golden):
    g = golden["replicate"]
    for j in range(5):
        L, step, shard, seed = (int(x) for x in g[f"rand_cfg_{j}"])
        rep = Rep(scheme=RANDOM, compression=float(g[f"rand_c_{j}"][0]), seed=seed)
        assert eq(oracle.selected_indices(rep, step, shard, L), g[f"rand_idx_{j}"]), j


def test_golden_optim_trajectories(oracle, golden):
    g = golden["optim"]
    rep = Rep(scheme=DEMO, chunk_size=64, top_k=32, compression=0.5, sign_mode=True, seed=1234)
    p = g["sgd_p0"].copy()
    m = np.zeros_like(p)
    for step in range(4):
        e = oracle.demo_sgd_prepare(m, g[f"sgd_g_{step}"], 0.9, rep, step, 0)
        for key in ("freq_indices", "values", "local_q", "m_accum", "m_after"):
            assert eq(e[key], g[f"sgd_{key}_{step}"]), (step, key)
        q = oracle.decode_and_merge(rep, [e["values"]], [e["freq_indices"]], len(p), step, 0)
        assert eq(q, g[f"sgd_q_{step}"])
        oracle.demo_sgd_apply(p, q, 0.01)
        assert eq(p, g[f"sgd_p_{step}"])
    rep = Rep(scheme=DEMO, chunk_size=64, top_k=16, compression=0.25, sign_mode=True, seed=1234)
    p = g["adam_p0"].copy()
    ea, es, steps = np.zeros_like(p), np.zeros_like(p), 0
    for step in range(4):
        gr = g[f"adam_g_{step}"]
        e = oracle.select_and_encode(gr, rep, step, 0)
        assert eq(e["freq_indices"], g[f"adam_idx_{step}"]) and eq(e["local_q"], g[f"adam_lq_{step}"])
        q = oracle.decode_and_merge(rep, [e["values"]], [e["freq_indices"]], len(p), step, 0)
        steps = oracle.adamw_apply(p, ea, es, steps, gr, e["local_q"], q, 0.9, 0.999, 1e-8, 0.01, 0.003)
        assert eq(p, g[f"adam_p_{step}"]) and eq(ea, g[f"adam_ea_{step}"]) and eq(es, g[f"adam_es_{step}"])
    out = oracle.grad_reduce_scatter([x.astype(np.float64) for x in g["rs_in"]])
    assert eq(out, g["rs_out"])


# ---------------------------------------------------------------- differential
@pytest.mark.skipif(reference() is None, reason="oracle/_ref not built (no /root/reference here)")
@pytest.mark.parametrize("seed", range(6))
def test_restatement_matches_reference_randomized(oracle, seed):
    ref = reference()
    rng = np.random.default_rng(seed)
    for _ in range(8):
        s = int(rng.choice([1, 2, 3, 7, 8, 16, 32, 64, 100, 128]))
        k = int(rng.integers(1, s + 1))
        n = int(rng.integers(1, 700))
        scheme = int(rng.choice([DEMO, RANDOM, STRIDING, DILOCO, FULL]))
        c = 1.0 if scheme == FULL else float(rng.choice([1 / 2, 1 / 4, 1 / 8, 1 / 3]))
        rep = Rep(scheme=scheme, chunk_size=s, top_k=k, compression=c, sign_mode=bool(rng.integers(2)),
                  transfer_dtype=int(rng.integers(3)), seed=int(rng.integers(1 << 40)))
        v = rng.standard_normal(n) * 10.0 ** rng.uniform(-6, 3, size=n)
        v[rng.random(n) < 0.05] = 0.0
        step, shard = int(rng.integers(50)), int(rng.integers(8))
        try:
            a = oracle.select_and_encode(v, rep, step, shard)
        except OracleError as e:
            with pytest.raises(OracleError) as e2:
                ref.select_and_encode(v, rep, step, shard)
            assert e2.value.code == e.code
            continue
        b = ref.select_and_encode(v, rep, step, shard)
        for key in a:
            assert np.array_equal(np.asarray(a[key]), np.asarray(b[key])), key
