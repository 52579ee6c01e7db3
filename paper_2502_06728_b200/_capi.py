"""ctypes binding of the C-ABI in include/demo_b200.h (libdemo_b200.so, in-tree).

The product path has no fallback: if the library is missing or cannot be
loaded this module raises ImportError at import time.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# DMB_LIB selects another build of the same library (tools/kernel_timeline.py loads the one
# compiled with -DDMB_KERNEL_EVENTS); it is never a CPU substitute
LIB_PATH = os.environ.get("DMB_LIB") or os.path.join(HERE, "libdemo_b200.so")

DMB_OK, DMB_TRAINING, DMB_CONFIG, DMB_PROTOCOL, DMB_CUDA = 0, 1, 2, 3, 4
ABI_VERSION = 1


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


class OptCfg(C.Structure):
    _fields_ = [
        ("kind", C.c_int32),
        ("_pad", C.c_int32),
        ("learning_rate", C.c_double),
        ("momentum_decay", C.c_double),
        ("adam_beta1", C.c_double),
        ("adam_beta2", C.c_double),
        ("adam_eps", C.c_double),
        ("weight_decay", C.c_double),
    ]


class ToyModel(C.Structure):
    """dmb_toy_model (model.hpp:36-46)"""
    _fields_ = [("kind", C.c_uint32), ("activation", C.c_uint32), ("loss", C.c_uint32), ("n_dims", C.c_uint32),
                ("dims", C.c_uint32 * 9)]


class ToyPool(C.Structure):
    """dmb_toy_pool: a dataset split resident on the device"""
    _fields_ = [("inputs", C.c_void_p), ("targets", C.c_void_p), ("labels", C.c_void_p), ("size", C.c_uint64)]


class Update(C.Structure):
    _fields_ = [
        ("scheme", C.c_int32),
        ("empty", C.c_int32),
        ("step", C.c_uint64),
        ("shard_id", C.c_uint32),
        ("wire_format", C.c_uint32),
        ("length", C.c_uint64),
        ("chunk_size", C.c_uint64),
        ("top_k", C.c_uint64),
        ("n_values", C.c_uint64),
        ("n_indices", C.c_uint64),
        ("bytes", C.c_uint64),
        ("body", C.c_void_p),
    ]


P = C.c_void_p
U64 = C.c_uint64
U32 = C.c_uint32
I32 = C.c_int32
D = C.c_double
PCFG = C.POINTER(RepCfg)
POPT = C.POINTER(OptCfg)
PUPD = C.POINTER(Update)
PU64 = C.POINTER(C.c_uint64)

_SIGS = {
    "dmb_abi_version": (C.c_int, []),
    "dmb_last_error": (C.c_char_p, []),
    "dmb_ctx_create": (C.c_int, [C.c_int, C.POINTER(P)]),
    "dmb_ctx_destroy": (C.c_int, [P]),
    "dmb_wire_bytes": (U64, [U64, U64, I32]),
    "dmb_period": (U64, [D]),
    "dmb_plan_update": (C.c_int, [PCFG, U64, U64, U32, PUPD]),
    "dmb_update_capacity": (U64, [PCFG, U64]),
    "dmb_selected_indices": (C.c_int, [P, PCFG, U64, U32, U64, P, PU64, P]),
    "dmb_select_and_encode": (C.c_int, [P, P, U64, PCFG, U64, U32, PUPD, P, P]),
    "dmb_decode_and_merge": (C.c_int, [P, PUPD, U64, PCFG, P, P]),
    "dmb_serialize": (C.c_int, [PUPD, I32, P, U64, PU64, P]),
    "dmb_deserialize": (C.c_int, [P, U64, I32, PUPD, PUPD, P]),
    "dmb_update_values": (C.c_int, [PUPD, I32, P, P]),
    "dmb_demo_sgd_prepare": (C.c_int, [P, P, P, P, U64, POPT, PCFG, U64, U32, PUPD, P, P, P]),
    "dmb_demo_sgd_apply": (C.c_int, [P, P, P, U64, D, P]),
    "dmb_adamw_prepare": (C.c_int, [P, P, U64, PCFG, U64, U32, PUPD, P, P]),
    "dmb_adamw_apply": (C.c_int, [P, P, P, P, PU64, P, P, P, U64, POPT, D, P]),
    "dmb_baseline_sgd_step": (C.c_int, [P, P, P, P, U64, POPT, D, P]),
    "dmb_merge_apply_sgd": (C.c_int, [P, PUPD, U64, PCFG, P, P, U64, U64, D, P]),
    "dmb_merge_apply_adamw": (C.c_int, [P, PUPD, U64, U64, PCFG, P, P, P, PU64, P, U64, U64, POPT, D, P]),
    "dmb_step_sgd_local": (C.c_int, [P, P, P, P, P, P, U64, POPT, PCFG, U64, U32, D, PUPD, P]),
    "dmb_step_adamw_local": (C.c_int, [P, P, P, P, P, P, P, P, PU64, U64, POPT, PCFG, U64, U32, D, PUPD, P]),
    "dmb_grad_mean": (C.c_int, [P, P, U64, U64, P, P]),
    "dmb_require_finite": (C.c_int, [P, P, U64, P]),
    "dmb_status": (C.c_int, [P, P, C.POINTER(C.c_int64)]),
    "dmb_fallback_chunks": (C.c_int, [P, P, PU64]),
    "dmb_launch_count": (U64, [P]),
    "dmb_set_wire_format": (C.c_int, [P, C.c_int32]),
    "dmb_plan_exchange": (C.c_int, [P, PCFG, U64, U64, U32, PUPD]),
    "dmb_chunk_layout": (C.c_int, [U64, U64, P]),
    "dmb_chunk": (C.c_int, [P, P, P, P, P]),
    "dmb_unchunk": (C.c_int, [P, P, P, P, P]),
    "dmb_dct2": (C.c_int, [P, P, U64, U64, P, P]),
    "dmb_idct3": (C.c_int, [P, P, U64, U64, P, P]),
    "dmb_extract_fast_components": (C.c_int, [P, P, U64, U64, U64, P, P, P, P, P]),
    "dmb_sign_transform": (C.c_int, [P, P, U64, P]),
    "dmb_grad_mean_pull": (C.c_int, [P, P, U64, U64, P, C.c_uint32, P]),
    "dmb_merge_apply_sgd_to": (C.c_int, [P, P, U64, P, P, P, U64, U64, C.c_double, P]),
    "dmb_merge_apply_adamw_to": (C.c_int, [P, P, U64, U64, P, P, P, P, P, P, P, P, P, U64, U64, P, C.c_double, P]),
    "dmb_set_sm_reserve": (C.c_int, [C.c_int]),
    "dmb_demo_sgd_prepare_members": (C.c_int, [P, P, C.c_uint32, P, P, P, U64, P, P, U64, C.c_uint32, P, P]),
    "dmb_step_sgd_local_members": (C.c_int, [P, P, C.c_uint32, P, P, P, P, P, U64, P, P, U64, C.c_uint32,
                                             C.c_double, P, P]),
    "dmb_adamw_prepare_members": (C.c_int, [P, P, C.c_uint32, P, U64, P, U64, C.c_uint32, P, P]),
    "dmb_step_adamw_local_members": (C.c_int, [P, P, C.c_uint32, P, P, P, P, P, P, P, P, U64, P, P, U64,
                                               C.c_uint32, C.c_double, P, P]),
    "dmb_toy_loss_grad": (C.c_int, [P, P, P, P, U64, U64, P, U64, U64, U64, P, U64, P, P]),
    "dmb_toy_loss": (C.c_int, [P, P, P, P, P, P]),
    "dmb_latch_export": (C.c_int, [P, P, P]),
    "dmb_latch_import": (C.c_int, [P, P, P]),
    "dmb_kernel_timer_enable": (C.c_int, [C.c_int]),
    "dmb_kernel_timer_read": (C.c_int, [C.POINTER(C.c_double), PU64]),
}

EXPORTED = tuple(_SIGS)


def load(path: str = LIB_PATH) -> C.CDLL:
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is missing: build the CUDA extension first "
            "(python -c 'import __graft_entry__ as g; g.build()' or make -C paper_2502_06728_b200/csrc)")
    lib = C.CDLL(path)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.dmb_abi_version() != ABI_VERSION:
        raise ImportError(f"{path}: ABI version {lib.dmb_abi_version()} != {ABI_VERSION}")
    return lib


lib = load()
