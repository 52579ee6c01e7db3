"""The transform.hpp:13-74 surface through the C ABI (dmb_chunk_layout / chunk / unchunk /
dct2 / idct3 / extract_fast_components / sign_transform) against the oracle and the golden
vectors of the reference build.  The DCTs accumulate in FP64 in the reference's order, so on
FP32 inputs they equal the oracle's FP64 result rounded to FP32, bit for bit."""
import numpy as np
import pytest
import torch

from oracle.oracle import DEMO, Rep

pytestmark = pytest.mark.gpu


def P():
    import paper_2502_06728_b200 as mod

    return mod


def f32(x):
    return np.asarray(x, np.float64).astype(np.float32)


@pytest.mark.parametrize("size,count", [(1, 3), (8, 5), (64, 100), (100, 7), (256, 3), (1024, 2)])
def test_dct2_idct3_bit_exact_after_rounding(oracle, size, count):
    p = P()
    rng = np.random.default_rng(size)
    x = rng.standard_normal((count, size)).astype(np.float32)
    x[0, : size // 2] = 0.0  # zero coefficients are skipped by the inverse (transform.cpp:69)
    B = oracle.dct_basis(size)
    xd = torch.from_numpy(x).cuda()
    got_f = p.dct2(xd).cpu().numpy()
    got_i = p.idct3(xd).cpu().numpy()
    for r in range(count):
        want_f = np.zeros(size)
        for j in range(size):  # acc = 0; acc += B[j][i] x[i], ascending i (transform.cpp:56-63)
            acc = 0.0
            for i in range(size):
                acc = acc + B[j, i] * float(x[r, i])
            want_f[j] = acc
        want_i = np.zeros(size)
        for j in range(size):  # ascending j, zeros skipped (transform.cpp:65-73)
            c = float(x[r, j])
            if c != 0.0:
                want_i = want_i + c * B[j]
        assert np.array_equal(got_f[r], f32(want_f)), r
        assert np.array_equal(got_i[r], f32(want_i)), r
        if size > 128:
            break  # the Python double loop is slow; one row is the bit-exact check


def test_chunk_unchunk_and_layout():
    p = P()
    lay = p.chunk_layout(100, 32)
    assert (lay.num_chunks, lay.pad) == (4, 28)
    with pytest.raises(p.ConfigError):
        p.chunk_layout(10, 0)
    v = torch.arange(100, dtype=torch.float32, device="cuda")
    rows = p.chunk(v, lay)
    assert rows.numel() == 128 and torch.equal(rows[:100], v) and not rows[100:].any()
    assert torch.equal(p.unchunk(rows, lay), v)
    with pytest.raises(p.ConfigError):
        p.chunk(v[:99], lay)


def test_sign_transform():
    p = P()
    v = torch.tensor([1.5, -2.0, 0.0, -0.0, float("nan"), 1e-30, -1e-30], device="cuda")
    p.sign_transform(v)
    assert v.cpu().tolist()[:4] == [1.0, -1.0, 0.0, 0.0]
    assert v.cpu().tolist()[4:] == [0.0, 1.0, -1.0]  # NaN -> 0 (transform.cpp:157-161)


def test_extract_fast_components_matches_golden(golden):
    p = P()
    g = golden["transform"]
    for ci in range(10):
        s, k, n = (int(x) for x in g[f"x_{ci}"])
        v = torch.from_numpy(g[f"v_{ci}"].astype(np.float32)).cuda()
        ex = p.extract_fast_components(v, s, k)
        assert np.array_equal(ex.selection.indices.cpu().numpy().astype(np.uint32), g[f"idx_{ci}"]), ci
        assert ex.selection.layout.num_chunks == (n + s - 1) // s
        co = ex.selection.coeffs.cpu().numpy().astype(np.float64)
        want = g[f"co_{ci}"]
        scale = np.maximum(np.abs(want).reshape(-1, k).max(axis=1), 1e-30).repeat(k)
        assert np.all(np.abs(co - want) <= 1e-5 * scale), ci
        fast = ex.fast.cpu().numpy().astype(np.float64)
        res = ex.residual.cpu().numpy().astype(np.float64)
        if k == s:  # full band: exact copy, zero residual (transform.cpp:119-125, :148-149)
            assert np.array_equal(fast, g[f"v_{ci}"].astype(np.float32).astype(np.float64))
            assert not res.any()
        else:
            assert np.array_equal(res, (v.cpu().numpy() - ex.fast.cpu().numpy()).astype(np.float64))
    with pytest.raises(p.ConfigError):
        p.extract_fast_components(torch.zeros(64, device="cuda"), 64, 65)
