"""CPU-side checks of the C-ABI boundary: the library loads, exports every symbol
include/demo_b200.h declares, and the host-only entry points (planning /
validation / byte model) follow the reference's rules.  No device work here."""
import ctypes as C
import os
import re

import pytest

from oracle.oracle import Rep

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_declared_symbol():
    from paper_2502_06728_b200 import _capi

    header = open(os.path.join(ROOT, "include", "demo_b200.h")).read()
    declared = set(re.findall(r"\b(dmb_[a-z0-9_]+)\s*\(", header))
    assert declared, "no declarations parsed"
    lib = C.CDLL(_capi.LIB_PATH)
    missing = [s for s in sorted(declared) if not hasattr(lib, s)]
    assert not missing, missing
    assert declared == set(_capi.EXPORTED), declared ^ set(_capi.EXPORTED)


def test_library_is_sm100a():
    from paper_2502_06728_b200 import _capi
    import subprocess

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _capi.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out, out


def test_wire_bytes_and_period_match_oracle(oracle):
    import paper_2502_06728_b200 as P

    for nv, ni in ((100, 0), (3, 0), (16, 16), (0, 0), (100, 100), (1600, 0), (12345, 77)):
        for d in (0, 1, 2):
            assert P.wire_bytes(nv, ni, d) == oracle.wire_bytes(nv, ni, d)
    for c in (0.125, 1 / 3, 1.0, 2.0, 1 / 16, 0.3, 1e-3):
        assert P.ReplicatorConfig(compression=c).period() == oracle.period(c)


def test_plan_update_headers_match_oracle(oracle):
    import paper_2502_06728_b200 as P

    for scheme in (1, 2, 3, 4, 5):
        for dtype in (0, 1, 2):
            for n in (1, 63, 64, 300, 4097):
                for step in (0, 1, 4, 7):
                    rep = Rep(scheme=scheme, chunk_size=64, top_k=8, compression=1.0 if scheme == 5 else 0.25,
                              sign_mode=True, transfer_dtype=dtype, seed=5)
                    cfg = P.ReplicatorConfig(P.Scheme(scheme), 64, 8, rep.compression, True, P.TransferDtype(dtype), 5)
                    try:
                        want = oracle.select_and_encode([1.0] * n, rep, step, 0)
                    except Exception:
                        with pytest.raises(P.ConfigError):
                            P.plan_update(cfg, n, step, 0)
                        continue
                    h = P.plan_update(cfg, n, step, 0)
                    assert h.bytes == want["bytes"] and bool(h.empty) == want["empty"]
                    assert h.n_values == len(want["values"]) and h.n_indices == len(want["freq_indices"])


def test_config_errors():
    import paper_2502_06728_b200 as P

    with pytest.raises(P.ConfigError, match="top_k"):
        P.plan_update(P.ReplicatorConfig(P.Scheme.DeMo, 32, 33), 100, 0, 0)
    with pytest.raises(P.ConfigError, match="top_k"):
        P.plan_update(P.ReplicatorConfig(P.Scheme.DeMo, 32, 0), 100, 0, 0)
    with pytest.raises(P.ConfigError, match="chunk size"):
        P.plan_update(P.ReplicatorConfig(P.Scheme.DeMo, 0, 1), 100, 0, 0)
    with pytest.raises(P.ConfigError, match="selects no components"):
        P.plan_update(P.ReplicatorConfig(P.Scheme.Random, compression=1e-6), 100, 0, 0)
    with pytest.raises(P.ConfigError, match="stride period"):
        P.plan_update(P.ReplicatorConfig(P.Scheme.Striding, compression=0.25), 3, 0, 0)


def test_sort16_network():
    """The select warps' 16-input sorting network (demo_tc_adam.cu, DMB_SORT16_NET) sorts
    every 0-1 input, hence every input (0-1 principle)."""
    import numpy as np

    src = open(os.path.join(ROOT, "paper_2502_06728_b200", "csrc", "demo_tc_adam.cu")).read()
    body = src[src.index("#define DMB_SORT16_NET(X)"):src.index("__device__ __forceinline__ void sort16_desc")]
    pairs = [(int(i), int(j)) for i, j in re.findall(r"X\((\d+), (\d+)\)", body)]
    assert len(pairs) == 60
    x = ((np.arange(1 << 16)[:, None] >> np.arange(16)) & 1).astype(np.int8)
    for i, j in pairs:
        hi, lo = np.maximum(x[:, i], x[:, j]), np.minimum(x[:, i], x[:, j])
        x[:, i], x[:, j] = hi, lo
    assert (np.diff(x, axis=1) <= 0).all()


@pytest.mark.parametrize("seed,block", [(12345, 1), (12345, 2), (987654321, 3), (2**63 + 5, 7), (1, 11)])
def test_mt19937_64_jump_ahead_is_exact(seed, block):
    """The Random scheme's substreams (random_index.cu): the start window of substream b, from
    the jump polynomial x^(b W) mod phi (phi by Berlekamp-Massey) correlated with the seeded
    engine's first words, equals the engine advanced b W outputs one by one (the first
    word up to its 31 low bits, never read by the twist), and the next 312 outputs match."""
    import ctypes as C

    from paper_2502_06728_b200 import _capi

    f = _capi.lib.dmb_debug_mt_jump_check
    f.argtypes = [C.c_uint64, C.c_uint64]
    f.restype = C.c_int
    assert f(seed, block) == 0
