"""Host-side mirror of the reference's optimizer / replication API (demosim core,
proj/core/include/demosim/{replicate,optim,transform}.hpp) over CUDA tensors.

Same names, argument meaning and error behaviour as the reference:
ConfigError / ProtocolError / TrainingError (common.hpp:10-26).  Vectors are
torch.float32 CUDA tensors instead of std::vector<double>; every computation
runs in libdemo_b200.so (include/demo_b200.h).  There is no CPU path.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import Optional, Sequence

import torch

from . import _capi
from ._capi import lib


class DemoError(RuntimeError):
    pass


class ConfigError(DemoError):
    """common.hpp:10-14"""


class ProtocolError(DemoError):
    """common.hpp:16-20"""


class TrainingError(DemoError):
    """common.hpp:22-26"""


class CudaError(DemoError):
    pass


_ERRORS = {1: TrainingError, 2: ConfigError, 3: ProtocolError, 4: CudaError}


def _check(rc: int):
    if rc != _capi.DMB_OK:
        raise _ERRORS.get(rc, DemoError)(lib.dmb_last_error().decode())


class Scheme(enum.IntEnum):
    """replicate.hpp:14 (the values are the wire tags)."""
    DeMo = 1
    Random = 2
    Striding = 3
    DiLoCo = 4
    Full = 5


class TransferDtype(enum.IntEnum):
    """replicate.hpp:16"""
    Fp32 = 0
    Fp16 = 1
    Ternary = 2


class OptimizerKind(enum.IntEnum):
    """optim.hpp:11"""
    DemoSgd = 0
    DecoupledAdamW = 1


@dataclass
class ReplicatorConfig:
    """replicate.hpp:28-39 (same defaults)."""
    scheme: Scheme = Scheme.DeMo
    chunk_size: int = 32
    top_k: int = 4
    compression: float = 0.125
    sign_mode: bool = True
    transfer_dtype: TransferDtype = TransferDtype.Fp32
    seed: int = 0

    def period(self) -> int:
        return int(lib.dmb_period(float(self.compression)))

    def c(self) -> _capi.RepCfg:
        return _capi.RepCfg(int(self.scheme), int(bool(self.sign_mode)), int(self.transfer_dtype), 0,
                            int(self.chunk_size), int(self.top_k), float(self.compression),
                            int(self.seed) & (2**64 - 1))


@dataclass
class OptimizerConfig:
    """optim.hpp:13-21 (same defaults)."""
    kind: OptimizerKind = OptimizerKind.DemoSgd
    learning_rate: float = 0.05
    momentum_decay: float = 0.9
    adam_beta1: float = 0.9
    adam_beta2: float = 0.999
    adam_eps: float = 1e-8
    weight_decay: float = 0.0

    def c(self) -> _capi.OptCfg:
        return _capi.OptCfg(int(self.kind), 0, self.learning_rate, self.momentum_decay, self.adam_beta1,
                            self.adam_beta2, self.adam_eps, self.weight_decay)


def wire_bytes(n_values: int, n_indices: int, dtype: TransferDtype) -> int:
    """replicate.hpp:24-26"""
    return int(lib.dmb_wire_bytes(n_values, n_indices, int(dtype)))


def value_bits(dtype: TransferDtype) -> int:
    """replicate.hpp:21-22"""
    return {TransferDtype.Fp32: 32, TransferDtype.Fp16: 16, TransferDtype.Ternary: 2}[TransferDtype(dtype)]


# ---------------------------------------------------------------- device context
class Context:
    """One dmb_ctx per device (basis tables, status latch, Random scratch)."""

    def __init__(self, device: int):
        self.device = device
        h = C.c_void_p()
        with torch.cuda.device(device):
            _check(lib.dmb_ctx_create(device, C.byref(h)))
        self.h = h

    def __del__(self):
        try:
            if self.h:
                lib.dmb_ctx_destroy(self.h)
        except Exception:
            pass


_contexts: dict = {}


def context(device=None) -> Context:
    dev = torch.cuda.current_device() if device is None else torch.device(device).index or 0
    if dev not in _contexts:
        _contexts[dev] = Context(dev)
    return _contexts[dev]


def _stream(t: Optional[torch.Tensor] = None):
    dev = t.device if t is not None else None
    return C.c_void_p(torch.cuda.current_stream(dev).cuda_stream)


def _ptr(t: Optional[torch.Tensor]):
    if t is None:
        return None
    return C.c_void_p(t.data_ptr())


def _vec(t: torch.Tensor, name: str) -> torch.Tensor:
    if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != torch.float32:
        raise ConfigError(f"{name} must be a float32 CUDA tensor")
    if not t.is_contiguous():
        raise ConfigError(f"{name} must be contiguous")
    return t


def status(device=None, stream=None) -> None:
    """Synchronize and raise TrainingError if a non-finite gradient was latched."""
    ctx = context(device)
    bad = C.c_int64(-1)
    _check(lib.dmb_status(ctx.h, stream or _stream(), C.byref(bad)))


def fallback_chunks(device=None) -> int:
    n = C.c_uint64(0)
    _check(lib.dmb_fallback_chunks(context(device).h, _stream(), C.byref(n)))
    return int(n.value)


def launch_count() -> int:
    return int(lib.dmb_launch_count(None))


# ---------------------------------------------------------------- CompressedUpdate
class CompressedUpdate:
    """replicate.hpp:43-59: header on the host, payload body on the device.  The body
    is byte-identical to the body of serialize() (replicate.cpp:316-356)."""

    def __init__(self, hdr: _capi.Update, body: Optional[torch.Tensor], dtype: TransferDtype):
        self.hdr = hdr
        self.body = body
        self.dtype = TransferDtype(dtype)
        if body is not None:
            self.hdr.body = body.data_ptr()

    scheme = property(lambda s: Scheme(s.hdr.scheme))
    step = property(lambda s: int(s.hdr.step))
    shard_id = property(lambda s: int(s.hdr.shard_id))
    length = property(lambda s: int(s.hdr.length))
    empty = property(lambda s: bool(s.hdr.empty))
    chunk_size = property(lambda s: int(s.hdr.chunk_size))
    top_k = property(lambda s: int(s.hdr.top_k))
    bytes = property(lambda s: int(s.hdr.bytes))

    def value_count(self) -> int:
        return int(self.hdr.n_values)

    @property
    def freq_indices(self) -> torch.Tensor:
        n = int(self.hdr.n_indices)
        if n == 0 or self.body is None:
            return torch.empty(0, dtype=torch.int32, device="cuda")
        return self.body[: 4 * n].view(torch.int32)

    @property
    def values(self) -> torch.Tensor:
        """Transmitted values at wire precision, as float32."""
        n = int(self.hdr.n_values)
        dev = self.body.device if self.body is not None else "cuda"
        out = torch.empty(n, dtype=torch.float32, device=dev)
        if n:
            _check(lib.dmb_update_values(C.byref(self.hdr), int(self.dtype), _ptr(out), _stream(out)))
        return out

    def with_header(self, **kw) -> "CompressedUpdate":
        """A copy sharing the body with some header fields replaced (protocol tests)."""
        h = _capi.Update.from_buffer_copy(self.hdr)
        for k, v in kw.items():
            setattr(h, k, v)
        u = CompressedUpdate(h, None, self.dtype)
        u.body = self.body
        return u


def _new_update(cfg: ReplicatorConfig, length: int, device) -> CompressedUpdate:
    c = cfg.c()
    cap = int(lib.dmb_update_capacity(C.byref(c), length))
    body = torch.empty(cap, dtype=torch.uint8, device=device)
    return CompressedUpdate(_capi.Update(), body, cfg.transfer_dtype)


@dataclass
class EncodeResult:
    """replicate.hpp:61-66"""
    update: CompressedUpdate
    local_q: Optional[torch.Tensor]


def plan_update(cfg: ReplicatorConfig, length: int, step: int, shard_id: int) -> _capi.Update:
    u = _capi.Update()
    c = cfg.c()
    _check(lib.dmb_plan_update(C.byref(c), length, step, shard_id, C.byref(u)))
    return u


def selected_indices(cfg: ReplicatorConfig, step: int, shard_id: int, length: int, device=None) -> torch.Tensor:
    """replicate.hpp:74-78: ascending uint32 index set (returned as int64)."""
    device = device or torch.device("cuda", torch.cuda.current_device())
    out = torch.empty(max(length, 1), dtype=torch.int32, device=device)
    n = C.c_uint64(0)
    c = cfg.c()
    _check(lib.dmb_selected_indices(context(device).h, C.byref(c), step, shard_id, length, _ptr(out),
                                    C.byref(n), _stream(out)))
    return out[: n.value].to(torch.int64) & 0xFFFFFFFF


def select_and_encode(v: torch.Tensor, cfg: ReplicatorConfig, step: int, shard_id: int) -> EncodeResult:
    """replicate.hpp:68-72"""
    _vec(v, "v")
    n = v.numel()
    upd = _new_update(cfg, n, v.device)
    lq = torch.empty_like(v)
    c = cfg.c()
    _check(lib.dmb_select_and_encode(context(v.device).h, _ptr(v), n, C.byref(c), step, shard_id,
                                     C.byref(upd.hdr), _ptr(lq), _stream(v)))
    return EncodeResult(upd, lq)


def _update_array(updates: Sequence[CompressedUpdate]):
    arr = (_capi.Update * max(len(updates), 1))()
    for i, u in enumerate(updates):
        arr[i] = u.hdr
    return arr


def decode_and_merge(updates: Sequence[CompressedUpdate], cfg: ReplicatorConfig) -> torch.Tensor:
    """replicate.hpp:80-84"""
    if not updates:
        raise ProtocolError("decode_and_merge needs at least one update")
    dev = next((u.body.device for u in updates if u.body is not None), torch.device("cuda"))
    q = torch.empty(updates[0].length, dtype=torch.float32, device=dev)
    arr = _update_array(updates)
    c = cfg.c()
    _check(lib.dmb_decode_and_merge(context(dev).h, arr, len(updates), C.byref(c), _ptr(q), _stream(q)))
    return q


def serialize(u: CompressedUpdate, dtype: TransferDtype) -> bytes:
    """replicate.hpp:86-88"""
    cap = 9 + u.bytes + 16
    buf = (C.c_uint8 * cap)()
    n = C.c_uint64(0)
    _check(lib.dmb_serialize(C.byref(u.hdr), int(dtype), buf, cap, C.byref(n), _stream()))
    return bytes(buf[: n.value])


def deserialize(buf: bytes, dtype: TransferDtype, shape_template: CompressedUpdate) -> CompressedUpdate:
    """replicate.hpp:90-93"""
    dev = shape_template.body.device if shape_template.body is not None else torch.device("cuda")
    body = torch.empty(max(len(buf), 16) + 16, dtype=torch.uint8, device=dev)
    out = CompressedUpdate(_capi.Update(), body, dtype)
    raw = (C.c_uint8 * max(len(buf), 1)).from_buffer_copy(buf if buf else b"\0")
    _check(lib.dmb_deserialize(raw, len(buf), int(dtype), C.byref(shape_template.hdr), C.byref(out.hdr),
                               _stream(body)))
    out.hdr.body = body.data_ptr()
    return out


# ---------------------------------------------------------------- optimizer
@dataclass
class MomentumState:
    """optim.hpp:23-31.  `m` is double buffered so a refused step leaves it untouched."""
    m: Optional[torch.Tensor] = None
    exp_avg: Optional[torch.Tensor] = None
    exp_avg_sq: Optional[torch.Tensor] = None
    steps: int = 0
    _spare: Optional[torch.Tensor] = field(default=None, repr=False)

    @staticmethod
    def make(kind: OptimizerKind, length: int, device=None) -> "MomentumState":
        device = device or torch.device("cuda", torch.cuda.current_device())
        st = MomentumState()
        if kind == OptimizerKind.DemoSgd:
            st.m = torch.zeros(length, dtype=torch.float32, device=device)
        else:
            st.exp_avg = torch.zeros(length, dtype=torch.float32, device=device)
            st.exp_avg_sq = torch.zeros(length, dtype=torch.float32, device=device)
        return st


@dataclass
class StepTrace:
    """optim.hpp:33-38"""
    m_accum: Optional[torch.Tensor] = None
    local_q: Optional[torch.Tensor] = None
    m_after: Optional[torch.Tensor] = None


def demo_sgd_prepare(state: MomentumState, grad: torch.Tensor, opt: OptimizerConfig, rep: ReplicatorConfig,
                     step: int, shard_id: int, trace: Optional[StepTrace] = None) -> EncodeResult:
    """optim.hpp:40-44"""
    _vec(grad, "grad")
    if state.m is None or grad.numel() != state.m.numel():
        raise ProtocolError("gradient and momentum lengths disagree")
    n = grad.numel()
    if state._spare is None or state._spare.numel() != n:
        state._spare = torch.empty_like(state.m)
    upd = _new_update(rep, n, grad.device)
    lq = torch.empty_like(grad)
    acc = torch.empty_like(grad) if trace is not None else None
    c, o = rep.c(), opt.c()
    ctx = context(grad.device)
    st = _stream(grad)
    _check(lib.dmb_demo_sgd_prepare(ctx.h, _ptr(grad), _ptr(state.m), _ptr(state._spare), n, C.byref(o),
                                    C.byref(c), step, shard_id, C.byref(upd.hdr), _ptr(lq), _ptr(acc), st))
    status(grad.device, st)  # require_finite (optim.cpp:21): raises before state changes
    state.m, state._spare = state._spare, state.m
    if trace is not None:
        trace.m_accum, trace.local_q, trace.m_after = acc, lq, state.m.clone()
    return EncodeResult(upd, lq)


def demo_sgd_apply(params: torch.Tensor, q: torch.Tensor, lr: float) -> None:
    """optim.hpp:46-48"""
    _vec(params, "params")
    _vec(q, "q")
    _check(lib.dmb_demo_sgd_apply(context(params.device).h, _ptr(params), _ptr(q), params.numel(), float(lr),
                                  _stream(params)))


def adamw_prepare(grad: torch.Tensor, rep: ReplicatorConfig, step: int, shard_id: int) -> EncodeResult:
    """optim.hpp:50-53"""
    _vec(grad, "grad")
    n = grad.numel()
    upd = _new_update(rep, n, grad.device)
    lq = torch.empty_like(grad)
    c = rep.c()
    st = _stream(grad)
    _check(lib.dmb_adamw_prepare(context(grad.device).h, _ptr(grad), n, C.byref(c), step, shard_id,
                                 C.byref(upd.hdr), _ptr(lq), st))
    status(grad.device, st)
    return EncodeResult(upd, lq)


def adamw_apply(params: torch.Tensor, state: MomentumState, grad: torch.Tensor, local_q: torch.Tensor,
                merged: Optional[torch.Tensor], opt: OptimizerConfig, lr: float) -> None:
    """optim.hpp:55-61"""
    for t, nm in ((params, "params"), (grad, "grad"), (local_q, "local_q")):
        _vec(t, nm)
    steps = C.c_uint64(state.steps)
    o = opt.c()
    _check(lib.dmb_adamw_apply(context(params.device).h, _ptr(params), _ptr(state.exp_avg), _ptr(state.exp_avg_sq),
                               C.byref(steps), _ptr(grad), _ptr(local_q), _ptr(merged), params.numel(), C.byref(o),
                               float(lr), _stream(params)))
    state.steps = int(steps.value)


def baseline_sgd_step(params: torch.Tensor, state: MomentumState, grad: torch.Tensor, opt: OptimizerConfig,
                      lr: float) -> None:
    """optim.hpp:66-67"""
    o = opt.c()
    st = _stream(params)
    _check(lib.dmb_baseline_sgd_step(context(params.device).h, _ptr(params), _ptr(state.m), _ptr(grad),
                                     params.numel(), C.byref(o), float(lr), st))
    status(params.device, st)


def baseline_adamw_step(params, state, grad, opt, lr) -> None:
    """optim.hpp:68-69 == adamw_apply(params, state, grad, grad, nullptr)"""
    st = _stream(params)
    o = opt.c()
    ctx = context(params.device)
    # require_finite first (optim.cpp:90), then the shared AdamW kernel
    _check(lib.dmb_require_finite(ctx.h, _ptr(grad), grad.numel(), st))
    status(params.device, st)
    steps = C.c_uint64(state.steps)
    _check(lib.dmb_adamw_apply(ctx.h, _ptr(params), _ptr(state.exp_avg), _ptr(state.exp_avg_sq), C.byref(steps),
                               _ptr(grad), _ptr(grad), None, params.numel(), C.byref(o), float(lr), st))
    state.steps = int(steps.value)


# ---------------------------------------------------------------- fused hot path
def merge_apply_sgd(updates: Sequence[CompressedUpdate], rep: ReplicatorConfig, params: torch.Tensor,
                    grad_if_unsynced: Optional[torch.Tensor], step: int, lr: float) -> None:
    """decode_and_merge + demo_sgd_apply without materializing Q (cluster.cpp:220-226)."""
    arr = _update_array(updates)
    c = rep.c()
    _check(lib.dmb_merge_apply_sgd(context(params.device).h, arr if updates else None, len(updates), C.byref(c),
                                   _ptr(params), _ptr(grad_if_unsynced), params.numel(), step, float(lr),
                                   _stream(params)))


def merge_apply_adamw(updates: Sequence[CompressedUpdate], own_rank: int, rep: ReplicatorConfig,
                      params: torch.Tensor, state: MomentumState, grad: torch.Tensor, step: int,
                      opt: OptimizerConfig, lr: float) -> None:
    """decode_and_merge + adamw_apply, local_q re-derived on the device (cluster.cpp:220-229)."""
    arr = _update_array(updates)
    c, o = rep.c(), opt.c()
    steps = C.c_uint64(state.steps)
    _check(lib.dmb_merge_apply_adamw(context(params.device).h, arr if updates else None, len(updates), own_rank,
                                     C.byref(c), _ptr(params), _ptr(state.exp_avg), _ptr(state.exp_avg_sq),
                                     C.byref(steps), _ptr(grad), params.numel(), step, C.byref(o), float(lr),
                                     _stream(params)))
    state.steps = int(steps.value)


def grad_mean(grads: Sequence[torch.Tensor]) -> torch.Tensor:
    """mean_of (vec.cpp:18-26): member-order elementwise mean on the device."""
    out = torch.empty_like(grads[0])
    arr = (C.c_void_p * len(grads))(*[g.data_ptr() for g in grads])
    _check(lib.dmb_grad_mean(context(out.device).h, arr, len(grads), out.numel(), _ptr(out), _stream(out)))
    return out


# ---------------------------------------------------------------- transform.hpp:13-74
@dataclass
class ChunkLayout:
    """transform.hpp:13-18"""
    length: int = 0
    chunk_size: int = 0
    num_chunks: int = 0
    pad: int = 0


class _Layout(C.Structure):
    _fields_ = [("length", C.c_uint64), ("chunk_size", C.c_uint64), ("num_chunks", C.c_uint64),
                ("pad", C.c_uint64)]


def chunk_layout(length: int, chunk_size: int) -> ChunkLayout:
    """transform.hpp:20 (ConfigError on chunk_size 0, transform.cpp:18)"""
    out = _Layout()
    _check(lib.dmb_chunk_layout(length, chunk_size, C.byref(out)))
    return ChunkLayout(out.length, out.chunk_size, out.num_chunks, out.pad)


def _layout_c(layout: ChunkLayout) -> _Layout:
    return _Layout(layout.length, layout.chunk_size, layout.num_chunks, layout.pad)


def chunk(v: torch.Tensor, layout: ChunkLayout) -> torch.Tensor:
    """transform.hpp:22-23: num_chunks x chunk_size rows, pad tail zeroed (flat)"""
    _vec(v, "v")
    if v.numel() != layout.length:
        raise ConfigError("chunk: layout does not match the vector")
    rows = torch.empty(layout.num_chunks * layout.chunk_size, dtype=torch.float32, device=v.device)
    lc = _layout_c(layout)
    _check(lib.dmb_chunk(context(v.device).h, _ptr(v), C.byref(lc), _ptr(rows), _stream(v)))
    return rows


def unchunk(rows: torch.Tensor, layout: ChunkLayout) -> torch.Tensor:
    """transform.hpp:25-26: concatenated rows without the pad tail"""
    _vec(rows, "rows")
    if rows.numel() != layout.num_chunks * layout.chunk_size:
        raise ConfigError("unchunk: row buffer does not match the layout")
    v = torch.empty(layout.length, dtype=torch.float32, device=rows.device)
    lc = _layout_c(layout)
    _check(lib.dmb_unchunk(context(rows.device).h, _ptr(rows), C.byref(lc), _ptr(v), _stream(rows)))
    return v


def _dct(x: torch.Tensor, inverse: bool) -> torch.Tensor:
    _vec(x, "x")
    size = x.shape[-1] if x.dim() > 1 else x.numel()
    count = x.numel() // size if size else 0
    out = torch.empty_like(x)
    f = lib.dmb_idct3 if inverse else lib.dmb_dct2
    _check(f(context(x.device).h, _ptr(x), size, count, _ptr(out), _stream(x)))
    return out


def dct2(x: torch.Tensor) -> torch.Tensor:
    """transform.hpp:51 (DctPlan::forward); a 2-D tensor transforms each row"""
    return _dct(x, False)


def idct3(coeffs: torch.Tensor) -> torch.Tensor:
    """transform.hpp:52 (DctPlan::inverse); a 2-D tensor transforms each row"""
    return _dct(coeffs, True)


@dataclass
class FreqSelection:
    """transform.hpp:55-62"""
    layout: ChunkLayout
    top_k: int
    indices: torch.Tensor  # int32 (uint32 values), num_chunks * top_k, chunk local, ascending
    coeffs: torch.Tensor


@dataclass
class Extraction:
    """transform.hpp:64-68"""
    selection: FreqSelection
    fast: torch.Tensor
    residual: torch.Tensor


def extract_fast_components(v: torch.Tensor, chunk_size: int, top_k: int) -> Extraction:
    """transform.hpp:70-71 / transform.cpp:94-155"""
    _vec(v, "v")
    layout = chunk_layout(v.numel(), chunk_size)
    n = layout.num_chunks * top_k if 1 <= top_k <= chunk_size else 0
    idx = torch.empty(max(n, 1), dtype=torch.int32, device=v.device)
    co = torch.empty(max(n, 1), dtype=torch.float32, device=v.device)
    fast, res = torch.empty_like(v), torch.empty_like(v)
    _check(lib.dmb_extract_fast_components(context(v.device).h, _ptr(v), v.numel(), chunk_size, top_k, _ptr(idx),
                                           _ptr(co), _ptr(fast), _ptr(res), _stream(v)))
    return Extraction(FreqSelection(layout, top_k, idx[:n], co[:n]), fast, res)


def sign_transform(v: torch.Tensor) -> None:
    """transform.hpp:73 (in place)"""
    _vec(v, "v")
    _check(lib.dmb_sign_transform(context(v.device).h, _ptr(v), v.numel(), _stream(v)))
