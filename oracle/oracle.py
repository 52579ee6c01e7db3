"""numpy face of the FP64 CPU oracles.  TEST INFRASTRUCTURE ONLY.

Two interchangeable libraries export the same ``dmo_*`` C symbols:

* ``restatement()`` -- oracle/demo_oracle.c, the committed C restatement of the
  reference path (built by oracle/Makefile into oracle/_build/);
* ``reference()``   -- the unmodified reference core compiled where it lies
  (oracle/_ref/libdemosim_ref.so; present only where /root/reference was).

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs import this module;
the product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
RESTATEMENT_SO = os.path.join(HERE, "_build", "libdemo_oracle.so")
REFERENCE_SO = os.path.join(HERE, "_ref", "libdemosim_ref.so")

DEMO, RANDOM, STRIDING, DILOCO, FULL = 1, 2, 3, 4, 5
FP32, FP16, TERNARY = 0, 1, 2
OK, TRAINING, CONFIG, PROTOCOL = 0, 1, 2, 3


class OracleError(Exception):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class RepCfg(C.Structure):
    _fields_ = [
        ("scheme", C.c_int32),
        ("sign_mode", C.c_int32),
        ("transfer_dtype", C.c_int32),
        ("_pad", C.c_int32),
        ("chunk_size", C.c_uint64),
        ("top_k", C.c_uint64),
        ("compression", C.c_double),
        ("seed", C.c_uint64),
    ]


@dataclass
class Rep:
    """Mirror of ReplicatorConfig (replicate.hpp:28-39) with the reference defaults."""

    scheme: int = DEMO
    chunk_size: int = 32
    top_k: int = 4
    compression: float = 0.125
    sign_mode: bool = True
    transfer_dtype: int = FP32
    seed: int = 0

    def c(self) -> RepCfg:
        return RepCfg(self.scheme, int(self.sign_mode), self.transfer_dtype, 0,
                      self.chunk_size, self.top_k, self.compression, self.seed)


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def build_restatement() -> str:
    if not os.path.exists(RESTATEMENT_SO) or os.path.getmtime(RESTATEMENT_SO) < max(
        os.path.getmtime(os.path.join(HERE, f)) for f in ("demo_oracle.c", "demo_oracle.h")
    ):
        subprocess.check_call(["make", "-s", "-C", HERE, "_build/libdemo_oracle.so"])
    return RESTATEMENT_SO


class Oracle:
    def __init__(self, path: str):
        self.path = path
        L = self.lib = C.CDLL(path)
        L.dmo_last_error.restype = C.c_char_p
        for name in ("dmo_mix_seed1", "dmo_mix_seed2", "dmo_mix_seed3"):
            getattr(L, name).restype = C.c_uint64
        L.dmo_mix_seed1.argtypes = [C.c_uint64]
        L.dmo_mix_seed2.argtypes = [C.c_uint64] * 2
        L.dmo_mix_seed3.argtypes = [C.c_uint64] * 3
        L.dmo_wire_bytes.restype = C.c_uint64
        L.dmo_wire_bytes.argtypes = [C.c_uint64, C.c_uint64, C.c_int]
        L.dmo_period.restype = C.c_uint64
        L.dmo_period.argtypes = [C.c_double]
        L.dmo_narrow_to_fp16.restype = C.c_double
        L.dmo_narrow_to_fp16.argtypes = [C.c_double]
        L.dmo_narrow_to_fp32.restype = C.c_double
        L.dmo_narrow_to_fp32.argtypes = [C.c_double]
        L.dmo_serialize.restype = C.c_uint64
        L.dmo_random_vector.argtypes = [C.c_uint64, C.c_size_t, C.c_void_p]
        L.dmo_mt64_stream.argtypes = [C.c_uint64, C.c_uint64, C.c_void_p]
        L.dmo_rng_below_batch.argtypes = [C.c_uint64, C.c_void_p, C.c_uint64, C.c_void_p]
        L.dmo_dct_basis.argtypes = [C.c_size_t, C.c_void_p]

    def _check(self, rc: int):
        if rc != OK:
            raise OracleError(rc, self.lib.dmo_last_error().decode())

    # ---- rng ---------------------------------------------------------------
    def mix_seed(self, *args) -> int:
        f = {1: self.lib.dmo_mix_seed1, 2: self.lib.dmo_mix_seed2, 3: self.lib.dmo_mix_seed3}
        return int(f[len(args)](*[C.c_uint64(a & (2**64 - 1)) for a in args]))

    def random_vector(self, seed: int, n: int) -> np.ndarray:
        out = np.empty(n, np.float64)
        self.lib.dmo_random_vector(C.c_uint64(seed), n, _p(out))
        return out

    def mt64_stream(self, seed: int, n: int) -> np.ndarray:
        out = np.empty(n, np.uint64)
        self.lib.dmo_mt64_stream(C.c_uint64(seed), n, _p(out))
        return out

    def rng_below(self, seed: int, ns) -> np.ndarray:
        ns = np.ascontiguousarray(ns, np.uint64)
        out = np.empty(len(ns), np.uint64)
        self.lib.dmo_rng_below_batch(C.c_uint64(seed), _p(ns), len(ns), _p(out))
        return out

    # ---- transform ----------------------------------------------------------
    def dct_basis(self, s: int) -> np.ndarray:
        b = np.empty(s * s, np.float64)
        self.lib.dmo_dct_basis(s, _p(b))
        return b.reshape(s, s)

    def extract(self, v, s: int, k: int):
        v = np.ascontiguousarray(v, np.float64)
        nc = (len(v) + s - 1) // s
        idx = np.empty(max(nc * k, 1), np.uint32)
        co = np.empty(max(nc * k, 1), np.float64)
        fast = np.empty(max(len(v), 1), np.float64)
        res = np.empty(max(len(v), 1), np.float64)
        self._check(self.lib.dmo_extract_fast_components(
            _p(v), C.c_size_t(len(v)), C.c_size_t(s), C.c_size_t(k), _p(idx), _p(co), _p(fast), _p(res)))
        return idx[: nc * k], co[: nc * k], fast[: len(v)], res[: len(v)]

    def sign_transform(self, v) -> np.ndarray:
        v = np.array(v, np.float64)
        self.lib.dmo_sign_transform(_p(v), C.c_size_t(len(v)))
        return v

    # ---- replicate --------------------------------------------------------
    def wire_bytes(self, nv: int, ni: int, dtype: int) -> int:
        return int(self.lib.dmo_wire_bytes(nv, ni, dtype))

    def period(self, c: float) -> int:
        return int(self.lib.dmo_period(c))

    def narrow_fp16(self, x: float) -> float:
        return float(self.lib.dmo_narrow_to_fp16(x))

    def narrow_fp32(self, x: float) -> float:
        return float(self.lib.dmo_narrow_to_fp32(x))

    def selected_indices(self, rep: Rep, step: int, shard: int, length: int) -> np.ndarray:
        out = np.empty(max(length, 1), np.uint32)
        cnt = C.c_uint64(0)
        cfg = rep.c()
        self._check(self.lib.dmo_selected_indices(C.byref(cfg), C.c_uint64(step), C.c_uint32(shard),
                                                  C.c_uint64(length), _p(out), C.byref(cnt)))
        return out[: cnt.value].copy()

    def _value_capacity(self, rep: Rep, length: int) -> int:
        if rep.scheme == DEMO:
            return ((length + rep.chunk_size - 1) // max(rep.chunk_size, 1)) * rep.top_k + 1
        return length + 1

    def select_and_encode(self, v, rep: Rep, step: int, shard: int) -> dict:
        v = np.ascontiguousarray(v, np.float64)
        n = len(v)
        cap = self._value_capacity(rep, n)
        idx = np.empty(cap, np.uint32)
        vals = np.empty(cap, np.float64)
        lq = np.empty(max(n, 1), np.float64)
        nv, ni, by = C.c_uint64(0), C.c_uint64(0), C.c_uint64(0)
        empty = C.c_int32(0)
        cfg = rep.c()
        self._check(self.lib.dmo_select_and_encode(
            _p(v), C.c_uint64(n), C.byref(cfg), C.c_uint64(step), C.c_uint32(shard), _p(idx), _p(vals),
            C.byref(nv), C.byref(ni), C.byref(by), C.byref(empty), _p(lq)))
        return dict(freq_indices=idx[: ni.value].copy(), values=vals[: nv.value].copy(),
                    bytes=by.value, empty=bool(empty.value), local_q=lq[:n].copy())

    def decode_and_merge(self, rep: Rep, values_list, idx_list, length: int, step: int, shard: int):
        R = len(values_list)
        vals = [np.ascontiguousarray(v, np.float64) for v in values_list]
        nv = len(vals[0]) if R else 0
        vp = (C.c_void_p * max(R, 1))(*[v.ctypes.data for v in vals])
        if rep.scheme == DEMO:
            idxs = [np.ascontiguousarray(i, np.uint32) for i in idx_list]
            ip = (C.c_void_p * max(R, 1))(*[i.ctypes.data for i in idxs])
        else:
            ip = (C.c_void_p * max(R, 1))()
        q = np.empty(max(length, 1), np.float64)
        cfg = rep.c()
        self._check(self.lib.dmo_decode_and_merge(
            C.byref(cfg), C.c_uint64(R), vp, ip, C.c_uint64(nv), C.c_uint64(length), C.c_uint64(step),
            C.c_uint32(shard), _p(q)))
        return q[:length].copy()

    def serialize(self, scheme: int, freq_indices, values, dtype: int) -> bytes:
        fi = np.ascontiguousarray(freq_indices if freq_indices is not None else [], np.uint32)
        va = np.ascontiguousarray(values, np.float64)
        out = np.empty(9 + 4 * len(fi) + 4 * len(va) + 8, np.uint8)
        n = self.lib.dmo_serialize(C.c_int(scheme), _p(fi), C.c_uint64(len(fi)), _p(va),
                                   C.c_uint64(len(va)), C.c_int(dtype), _p(out))
        return out[:n].tobytes()

    # ---- optim ------------------------------------------------------------
    def demo_sgd_prepare(self, m, grad, beta: float, rep: Rep, step: int, shard: int) -> dict:
        """Returns the encode result plus the StepTrace; `m` (np.float64) is updated in place."""
        g = np.ascontiguousarray(grad, np.float64)
        n = len(g)
        cap = self._value_capacity(rep, n)
        idx = np.empty(cap, np.uint32)
        vals = np.empty(cap, np.float64)
        lq = np.empty(max(n, 1), np.float64)
        acc = np.empty(max(n, 1), np.float64)
        nv, by = C.c_uint64(0), C.c_uint64(0)
        empty = C.c_int32(0)
        bad = C.c_int64(-1)
        cfg = rep.c()
        rc = self.lib.dmo_demo_sgd_prepare(
            _p(m), _p(g), C.c_uint64(n), C.c_double(beta), C.byref(cfg), C.c_uint64(step),
            C.c_uint32(shard), _p(idx), _p(vals), C.byref(nv), C.byref(by), C.byref(empty), _p(lq),
            _p(acc), C.byref(bad))
        self._check(rc)
        ni = nv.value if rep.scheme == DEMO else 0
        return dict(freq_indices=idx[:ni].copy(), values=vals[: nv.value].copy(), bytes=by.value,
                    empty=bool(empty.value), local_q=lq[:n].copy(), m_accum=acc[:n].copy(),
                    m_after=m.copy())

    def demo_sgd_apply(self, p, q, lr: float):
        self.lib.dmo_demo_sgd_apply(_p(p), _p(np.ascontiguousarray(q, np.float64)), C.c_uint64(len(p)),
                                    C.c_double(lr))

    def adamw_apply(self, p, exp_avg, exp_avg_sq, steps: int, grad, local_q, merged, beta1, beta2, eps,
                    wd, lr) -> int:
        st = C.c_uint64(steps)
        g = np.ascontiguousarray(grad, np.float64)
        lq = np.ascontiguousarray(local_q, np.float64)
        mg = None if merged is None else np.ascontiguousarray(merged, np.float64)
        self.lib.dmo_adamw_apply(_p(p), _p(exp_avg), _p(exp_avg_sq), C.byref(st), _p(g), _p(lq),
                                 None if mg is None else _p(mg), C.c_uint64(len(p)), C.c_double(beta1),
                                 C.c_double(beta2), C.c_double(eps), C.c_double(wd), C.c_double(lr))
        return st.value

    def grad_reduce_scatter(self, grads) -> np.ndarray:
        gs = [np.ascontiguousarray(g, np.float64) for g in grads]
        A, n = len(gs), len(gs[0])
        gp = (C.c_void_p * A)(*[g.ctypes.data for g in gs])
        out = np.empty(n, np.float64)
        self._check(self.lib.dmo_grad_reduce_scatter(C.c_uint64(A), C.c_uint64(n), gp, _p(out)))
        return out.reshape(A, n // A)


_cache: dict = {}


def restatement() -> Oracle:
    if "r" not in _cache:
        _cache["r"] = Oracle(build_restatement())
    return _cache["r"]


def reference() -> Oracle | None:
    """The unmodified reference build, or None where it was not built (GPU box)."""
    if "ref" not in _cache:
        _cache["ref"] = Oracle(REFERENCE_SO) if os.path.exists(REFERENCE_SO) else None
    return _cache["ref"]
