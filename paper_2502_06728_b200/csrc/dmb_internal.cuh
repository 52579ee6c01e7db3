// dmb_internal.cuh -- shared device helpers and launch interfaces of the
// B200-native FlexDeMo optimizer step (sm_100a only).
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "demo_b200.h"

namespace dmb {

// kernels launched through this library (the bench's gpu_launches evidence)
void count_launches(int n);
int sm_reserve();  // SMs the persistent step kernels leave free (dmb_set_sm_reserve)
// dmb_kernel_timer_*: events around the dominant tensor-core kernel's launches
void timer_begin(cudaStream_t stream);
void timer_end(cudaStream_t stream);

constexpr unsigned kFull = 0xffffffffu;
constexpr unsigned long long kNoBad = ~0ull;
constexpr int kMaxReplicas = 64;

// Device-side status latch (one per context).  first_bad follows
// require_finite (vec.cpp:7-16): the lowest non-finite gradient index wins.
struct DevStatus {
  unsigned long long first_bad;       // kNoBad when clean
  unsigned long long fallback_chunks; // FP64 re-derivations (certification misses)
  unsigned int protocol_error;        // frequency index out of range (replicate.cpp:293)
  unsigned int _pad;
};

// R replica bodies for a merge, passed by value (rank order == member order).
struct Bodies {
  const uint8_t* body[kMaxReplicas];
  int R;
};

// Wire-format value access (replicate.cpp:316-356 body layout).
__device__ __forceinline__ float load_wire_value(const uint8_t* vals, uint64_t t, int dtype) {
  if (dtype == DMB_FP32) return reinterpret_cast<const float*>(vals)[t];
  if (dtype == DMB_FP16) return __half2float(reinterpret_cast<const __half*>(vals)[t]);
  const uint32_t code = (vals[t >> 2] >> (2 * (t & 3))) & 3u;  // 1:+1 2:-1 0/3:0
  return code == 1u ? 1.0f : (code == 2u ? -1.0f : 0.0f);
}

// sign_transform (transform.cpp:157-161): x>0 -> 1, x<0 -> -1, else (0, -0, NaN) -> +0
__device__ __forceinline__ float sign_of(float x) {
  return x > 0.0f ? 1.0f : (x < 0.0f ? -1.0f : 0.0f);
}

// Wire store of an already conditioned value w (sign / fp16 rounding applied by
// condition_f32 or the FP64 path) at position t.  Ternary packs 2-bit codes with
// atomicOr into a pre-zeroed region (LSB first, replicate.cpp:340-352).
__device__ __forceinline__ void store_wire_value(uint8_t* vals, uint64_t t, float w, int dtype) {
  if (dtype == DMB_FP32) {
    reinterpret_cast<float*>(vals)[t] = w;
  } else if (dtype == DMB_FP16) {
    reinterpret_cast<__half*>(vals)[t] = __float2half_rn(w);
  } else {
    const uint32_t code = w > 0.0f ? 1u : (w < 0.0f ? 2u : 0u);
    if (code) atomicOr(reinterpret_cast<unsigned int*>(vals) + (t >> 4), code << (2 * (t & 15)));
  }
}

// condition_values (replicate.cpp:137-144) on an FP32 value
__device__ __forceinline__ float condition_f32(float c, int dtype, bool sign_mode) {
  if (sign_mode || dtype == DMB_TERNARY) return sign_of(c);
  if (dtype == DMB_FP16) return __half2float(__float2half_rn(c));
  return c;
}
// ... and on an FP64 coefficient (the certified-fallback path): one rounding only
__device__ __forceinline__ float condition_f64(double c, int dtype, bool sign_mode) {
  if (sign_mode || dtype == DMB_TERNARY) return c > 0.0 ? 1.0f : (c < 0.0 ? -1.0f : 0.0f);
  if (dtype == DMB_FP16) return __half2float(__double2half(c));
  return (float)c;
}

__device__ __forceinline__ void latch_bad(DevStatus* st, uint64_t index) {
  atomicMin(&st->first_bad, (unsigned long long)index);
}

__device__ __forceinline__ bool step_failed(const DevStatus* st) {
  return *(volatile const unsigned long long*)&st->first_bad != kNoBad;
}

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Step scalars computed on the host in double (optim.cpp:25, :62-63, :45).
struct SgdScalars {
  float beta;  // momentum_decay
  float lr;
};
struct AdamScalars {
  float beta1, one_minus_beta1, beta2, one_minus_beta2;
  float inv_bc1, inv_bc2;  // 1/(1 - beta^t), std::pow on the host (optim.cpp:62-63)
  float eps, lr, lr_wd;    // lr * weight_decay (0 disables, optim.cpp:71)
  float lr_bc1;            // lr / (1 - beta1^t)
};

// m_hat / (sqrt(v_hat) + eps), optim.cpp:68-70.  The IEEE sqrtf and '/' compile to a slow-path
// check, a CALL and a reconvergence point per element, which made this kernel 2.7x slower
// (measured: 19.6 ms against 7.2 ms per OLMo-1B step); the hardware square root and a
// Newton-refined reciprocal are each within a few ulp (~1e-7 relative), two orders below the
// 1e-5 parity bar -- the tests and smoke() print the error actually reached.
__device__ __forceinline__ float adam_ratio(float m1, float m2, const AdamScalars& A) {
  float sq, r;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(sq) : "f"(m2 * A.inv_bc2));
  const float d = sq + A.eps;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(d));
  r = fmaf(r, fmaf(-d, r, 1.0f), r);
  return (m1 * A.inv_bc1) * r;
}


// ---------------------------------------------------------------------------
// Kernel launch interfaces (implemented in demo_chunk.cu / sparse_schemes.cu /
// random_index.cu).  All take the launch stream last.

struct DemoGeometry {
  uint64_t len;        // shard length (real_len)
  uint64_t nchunks;    // ceil(len / s)
  int s, k;            // chunk_size, top_k
  int dtype;           // transfer dtype
  bool sign_mode;
  int wire_mask;       // DMB_WIRE_MASK bodies (tensor-core AdamW kernels only)
};
// MASK body: u64 masks, then values (2-bit codes when signs travel)
__device__ __forceinline__ int mask_value_dtype(const DemoGeometry& g) {
  return (g.sign_mode || g.dtype == DMB_TERNARY) ? DMB_TERNARY : g.dtype;
}

// Device basis tables for one chunk size (host-computed FP64 with libm cos,
// transform.cpp:41-54; FP32 copies are rounded from it).
struct Basis {
  int s;
  const float* B;    // [j][i] row-major, s*s
  const float* BT;   // [i][j] transposed
  const double* B64; // [j][i] row-major
  const double* B64T; // [i][j] transposed
  // TF32 splits for the tensor-core path (hi = RNA_tf32(B64), lo = RNA_tf32(B64 - hi))
  const float* Bhi;
  const float* Blo;
  const float* BThi;
  const float* BTlo;
};

enum class ChunkMode : int {
  EncodeSgd = 0,     // m_acc = beta m + g -> encode; m_out = m_acc - local_q
  EncodeAdam = 1,    // v = g -> encode (no state change)
  StepSgd = 2,       // EncodeSgd + merge(R=1) + p_out = p_in - lr Q
  StepAdam = 3,      // EncodeAdam + merge(R=1) + AdamW apply
  MergeSgd = 4,      // R bodies -> Q -> p_out = p_in - lr Q (Q optionally stored)
  MergeAdam = 5,     // R bodies -> Q; local_q from g + own indices -> AdamW apply
};

struct ChunkArgs {
  DemoGeometry geo;
  Basis basis;
  const float* g;
  const float* m_in;
  float* m_out;
  const float* p_in;
  float* p_out;
  const float* ea_in;
  float* ea_out;
  const float* es_in;
  float* es_out;
  float* local_q;   // nullable
  float* m_accum;   // nullable (StepTrace.m_accum)
  float* q_out;     // nullable (merged Q, decode_and_merge)
  uint8_t* body;    // own payload (nullable in Step* modes)
  Bodies in;        // merge inputs
  int own_rank;     // MergeAdam: which body is this rank's
  SgdScalars sgd;
  AdamScalars adam;
  DevStatus* status;
  // tensor-core path: chunks whose FP32 TopK is not certified go to this list and are
  // re-derived in FP64 by the SIMT kernel in list mode (list / list_count, force_fp64)
  uint32_t* fb_list;
  unsigned* fb_count;
  const uint32_t* list;
  const unsigned* list_count;
  int force_fp64;
  uint64_t first_chunk;     // SIMT kernel, non-list mode: start at this chunk (tail fix-up)
  unsigned long long* dbg;  // optional event timestamps (tests / tuning only)
  // the shard group's reduce-scatter fused into the gradient load (StepAdam / EncodeAdam on the
  // tensor-core kernel): the encoded gradient is the member-order mean of g_src[0..n_src), and
  // the kernel writes that mean to g (which every later reader -- fix-up, tail, merge -- uses)
  const float* g_src[4];
  int n_src;
};
constexpr int kMaxGradSrc = 4;

// Dispatch: tensor-core kernel + FP64 fix-up for s == 64 when enabled, else SIMT.
void launch_chunk_kernel(ChunkMode mode, const ChunkArgs& a, cudaStream_t stream);
void launch_chunk_simt(ChunkMode mode, const ChunkArgs& a, cudaStream_t stream);
bool tc_supported(ChunkMode mode, const ChunkArgs& a);
void launch_tc_kernel(ChunkMode mode, const ChunkArgs& a, cudaStream_t stream);
bool tc_enabled();
bool tc3_supported(ChunkMode mode, const ChunkArgs& a);
bool tc3_available();  // the tensor-map encoder of the driver is reachable
void launch_tc3_kernel(ChunkMode mode, const ChunkArgs& a, cudaStream_t stream);
// exact FP64 re-derivation of the full chunks listed in a.fb_list / a.fb_count
void launch_fix64_kernel(ChunkMode mode, const ChunkArgs& a, cudaStream_t stream);

// Elementwise (Full / DiLoCo / Striding / Random) paths.
struct SparseSel {
  int scheme;               // 0 (none), DMB_FULL, DMB_DILOCO, DMB_STRIDING, DMB_RANDOM
  uint64_t len;
  uint64_t offset, period;  // striding
  uint64_t count;           // number of selected values
  const uint32_t* bitmap;   // random: 1 bit per element
  const uint32_t* rank;     // random: selected count before each 32-bit word
};

void launch_sparse_encode(const SparseSel& sel, bool sgd, const float* g, const float* m_in,
                          float* m_out, float beta, float* local_q, float* m_accum,
                          uint8_t* vals, int dtype, bool sign_mode, DevStatus* st,
                          cudaStream_t stream);
void launch_sparse_merge_apply(const SparseSel& sel, const Bodies& in, int dtype, int mode,
                               const float* g, const float* p_in, float* p_out,
                               const float* ea_in, float* ea_out, const float* es_in,
                               float* es_out, float* q_out, SgdScalars sgd, AdamScalars adam,
                               DevStatus* st, cudaStream_t stream);
// mode for launch_sparse_merge_apply
enum { kMergeOnly = 0, kMergeSgd = 1, kMergeAdam = 2 };

void launch_sgd_apply(float* p, const float* q, uint64_t n, float lr, const DevStatus* st,
                      cudaStream_t stream);
void launch_adamw_apply(float* p, float* ea, float* es, const float* g, const float* lq,
                        const float* merged, uint64_t n, AdamScalars a, const DevStatus* st,
                        cudaStream_t stream);
void launch_baseline_sgd(float* p, float* m, const float* g, uint64_t n, float beta, float lr,
                         DevStatus* st, cudaStream_t stream);
void launch_check_finite(const float* g, uint64_t n, DevStatus* st, cudaStream_t stream);
void launch_grad_mean(const float* const* grads, int members, uint64_t n, float* out,
                      cudaStream_t stream);
void launch_grad_mean_pull(const float* const* grads, int members, uint64_t n, float* out, int ctas,
                           cudaStream_t stream);
void launch_striding_iota(uint32_t* out, uint64_t offset, uint64_t period, uint64_t count,
                          cudaStream_t stream);
void launch_unpack_values(const uint8_t* vals, uint64_t n, int dtype, float* out,
                          cudaStream_t stream);

// transform.hpp surface (transform.cu)
void launch_chunk(const float* v, uint64_t len, uint64_t padded, float* rows, cudaStream_t st);
void launch_copy(const float* a, uint64_t n, float* out, cudaStream_t st);
void launch_dct(bool inverse, const float* in, uint64_t n, uint64_t count, const Basis& b, float* out,
                cudaStream_t st);
void launch_sign(float* v, uint64_t n, cudaStream_t st);
void launch_residual(const float* v, const float* fast, uint64_t n, bool full_band, float* res, cudaStream_t st);

// toy gradient producers (toy_models.cu; model.cpp) for the trainer loop
constexpr int kToyMaxDims = 9;  // an input and up to 8 layers
struct ToyArgs {
  int kind;           // 0 quadratic, 1 mlp
  int activation;     // 0 tanh, 1 relu
  int loss_kind;      // 0 mse, 1 cross entropy
  uint32_t n_dims;
  uint32_t dims[kToyMaxDims];
  const double* inputs;    // pool x dims[0]
  const double* targets;   // pool x dims.back() (mse) or null
  const int32_t* labels;   // pool (cross entropy) or null
  const int64_t* order;    // BatchStream permutation, or null: examples 0..batch-1
  uint64_t order_len;
  uint64_t step, world, batch;
  const float* params;     // rows of params_stride; worker w reads row w / workers_per_row
  uint64_t params_stride, workers_per_row, workers;
  float* grad;             // workers x grad_stride, grad_len written (pad zeroed); null: loss only
  uint64_t grad_stride, grad_len;
  double* loss;            // workers
};
uint64_t toy_smem_bytes(const ToyArgs& a);
int launch_toy(const ToyArgs& a, cudaStream_t stream);

// Random index sets (replicate.cpp:160-172) on the device.
struct RandomScratch {
  uint32_t* draws;   // j_i for the L - count iterations that decide the set
  uint32_t* first;   // per position: smallest iteration that targeted it
  uint32_t* second;  // per position: second smallest
  uint32_t* bitmap;  // selected values, 1 bit each
  uint32_t* rank;    // exclusive prefix popcount per 32-bit word
  uint32_t* idx;     // sorted selected indices
  uint64_t capacity; // elements
  // MT19937-64 substreams (random_index.cu): the engine's first words, the start window of
  // every substream, the first output a Lemire rejection may touch
  uint64_t* mt_seq;
  uint64_t* mt_windows;
  uint64_t mt_blocks_cap;
  unsigned long long* mt_reject;
};
constexpr uint64_t kMtMaxSubstreams = 4096;           // substream windows held per context
constexpr uint64_t kMtSeqWords = 312ull * 65ull;       // seeded words + 64 twists (>= 19937 + 312)
// returns DMB_OK or DMB_CUDA (message in *err)
int launch_random_indices(uint64_t engine_seed, uint64_t len, uint64_t count, const RandomScratch& s,
                          cudaStream_t stream, const char** err);
// host-only check of the substream jump-ahead (tests): 0 when substream b's start window is exact
int mt_jump_check(uint64_t engine_seed, uint64_t b, const char** err);

}  // namespace dmb
