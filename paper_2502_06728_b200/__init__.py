"""B200-native FlexDeMo / DeToNATION optimizer step (arXiv 2502.06728).

Drop-in for the reference's optimizer and replication-scheme API (demosim core):
every computation runs in the sm_100a library libdemo_b200.so through the C-ABI
in include/demo_b200.h.  Importing this package fails loudly if the library is
missing -- there is no CPU fallback.
"""
from .core import (CompressedUpdate, ConfigError, CudaError, DemoError, EncodeResult, MomentumState,  # noqa: F401
                   OptimizerConfig, OptimizerKind, ProtocolError, ReplicatorConfig, Scheme, StepTrace,
                   TrainingError, TransferDtype, adamw_apply, adamw_prepare, baseline_adamw_step,
                   baseline_sgd_step, decode_and_merge, demo_sgd_apply, demo_sgd_prepare, deserialize,
                   fallback_chunks, grad_mean, launch_count, merge_apply_adamw, merge_apply_sgd, plan_update,
                   select_and_encode, selected_indices, serialize, status, value_bits, wire_bytes)
from .core import (ChunkLayout, Extraction, FreqSelection, chunk, chunk_layout, dct2,  # noqa: F401
                   extract_fast_components, idct3, sign_transform, unchunk)
from ._capi import LIB_PATH  # noqa: F401
