// sparse_schemes.cu -- Full / DiLoCo / Striding / Random encode + merge + apply,
// and the standalone elementwise optimizer kernels.  All HBM-bound: grid-stride
// loops sized to a multiple of the SM count, one element per thread-iteration,
// coalesced 4-byte accesses (the selected-value payload is indexed by rank).
//
//   select_and_encode (Full/DiLoCo/Random/Striding)  replicate.cpp:197-222
//   decode_and_merge  (Full/DiLoCo/Random/Striding)  replicate.cpp:260-281
//   demo_sgd_apply                                   optim.cpp:45-49
//   adamw_apply                                      optim.cpp:57-74
//   baseline_sgd_step                                optim.cpp:76-86
//   mean_of (grad_reduce_scatter's reduction)        vec.cpp:18-26
#include "dmb_internal.cuh"

namespace dmb {
namespace {

constexpr int kBlock = 256;

unsigned grid_for(uint64_t n, int per_sm = 8) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const uint64_t want = (n + kBlock - 1) / kBlock;
  const uint64_t cap = (uint64_t)sms * per_sm;
  return (unsigned)(want < cap ? (want ? want : 1) : cap);
}

// Is element i transmitted, and if so at which value slot?
__device__ __forceinline__ bool selected(const SparseSel& s, uint64_t i, uint64_t& slot) {
  switch (s.scheme) {
    case 0:  // nothing transmitted (DiLoCo between beats, replicate.cpp:202-207)
      return false;
    case DMB_FULL:
    case DMB_DILOCO:
      slot = i;
      return true;
    case DMB_STRIDING:
      if (i < s.offset || (i - s.offset) % s.period != 0) return false;
      slot = (i - s.offset) / s.period;
      return true;
    default: {  // random: bitmap + per-word rank
      const uint32_t w = s.bitmap[i >> 5];
      const uint32_t bit = 1u << (i & 31);
      if (!(w & bit)) return false;
      slot = s.rank[i >> 5] + __popc(w & (bit - 1));
      return true;
    }
  }
}

__global__ void sparse_encode_kernel(SparseSel sel, bool sgd, const float* __restrict__ g,
                                     const float* __restrict__ m_in, float* __restrict__ m_out,
                                     float beta, float* __restrict__ local_q,
                                     float* __restrict__ m_accum, uint8_t* __restrict__ vals,
                                     int dtype, bool sign_mode, DevStatus* st) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < sel.len; i += stride) {
    const float gi = g[i];
    if (!isfinite(gi)) latch_bad(st, i);
    const float x = sgd ? __fadd_rn(__fmul_rn(beta, m_in[i]), gi) : gi;  // optim.cpp:27
    if (m_accum) m_accum[i] = x;
    uint64_t slot;
    const bool on = selected(sel, i, slot);
    if (on && vals) store_wire_value(vals, slot, condition_f32(x, dtype, sign_mode), dtype);
    if (local_q) local_q[i] = on ? x : 0.0f;
    if (sgd) m_out[i] = on ? x - x : x;  // optim.cpp:35-37 with local_q = x or 0
  }
}

template <int MODE>
__global__ void sparse_merge_kernel(SparseSel sel, Bodies in, int dtype,
                                    const float* __restrict__ g, const float* __restrict__ p_in,
                                    float* __restrict__ p_out, const float* __restrict__ ea_in,
                                    float* __restrict__ ea_out, const float* __restrict__ es_in,
                                    float* __restrict__ es_out, float* __restrict__ q_out,
                                    SgdScalars sgd, AdamScalars A, DevStatus* st) {
  if (step_failed(st)) return;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const float R = (float)in.R;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < sel.len; i += stride) {
    uint64_t slot;
    const bool on = selected(sel, i, slot);
    float q = 0.0f;
    if (on) {
      float acc = 0.0f;  // member order (replicate.cpp:264-265, :277-279)
      for (int r = 0; r < in.R; ++r) acc += load_wire_value(in.body[r], slot, dtype);
      q = acc / R;
    }
    if (q_out) q_out[i] = q;
    if (MODE == kMergeSgd) {
      p_out[i] = p_in[i] - sgd.lr * q;
    } else if (MODE == kMergeAdam) {
      // g' = g - local_q + merged with local_q = g on selected slots, else 0
      const float gi = g[i];
      const float gp = on ? (gi - gi) + q : (gi - 0.0f) + q;
      const float ea = A.beta1 * ea_in[i] + A.one_minus_beta1 * gp;
      const float es = A.beta2 * es_in[i] + A.one_minus_beta2 * gp * gp;
      float p = p_in[i] - A.lr * ((ea * A.inv_bc1) / (sqrtf(es * A.inv_bc2) + A.eps));
      if (A.lr_wd != 0.0f) p -= A.lr_wd * p;
      ea_out[i] = ea;
      es_out[i] = es;
      p_out[i] = p;
    }
  }
}

__global__ void sgd_apply_kernel(float* __restrict__ p, const float* __restrict__ q, uint64_t n,
                                 float lr, const DevStatus* st) {
  if (step_failed(st)) return;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    p[i] = p[i] - lr * q[i];
}

__global__ void adamw_apply_kernel(float* __restrict__ p, float* __restrict__ ea_,
                                   float* __restrict__ es_, const float* __restrict__ g,
                                   const float* __restrict__ lq, const float* __restrict__ merged,
                                   uint64_t n, AdamScalars A, const DevStatus* st) {
  if (step_failed(st)) return;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const float gp = merged ? (g[i] - lq[i]) + merged[i] : g[i];
    const float ea = A.beta1 * ea_[i] + A.one_minus_beta1 * gp;
    const float es = A.beta2 * es_[i] + A.one_minus_beta2 * gp * gp;
    float pv = p[i] - A.lr * ((ea * A.inv_bc1) / (sqrtf(es * A.inv_bc2) + A.eps));
    if (A.lr_wd != 0.0f) pv -= A.lr_wd * pv;
    ea_[i] = ea;
    es_[i] = es;
    p[i] = pv;
  }
}

__global__ void baseline_sgd_kernel(float* __restrict__ p, float* __restrict__ m,
                                    const float* __restrict__ g, uint64_t n, float beta, float lr,
                                    const DevStatus* st) {
  if (step_failed(st)) return;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const float v = __fadd_rn(__fmul_rn(beta, m[i]), g[i]);
    p[i] = p[i] - lr * v;
    m[i] = 0.0f;
  }
}

__global__ void check_finite_kernel(const float* __restrict__ g, uint64_t n, DevStatus* st) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    if (!isfinite(g[i])) latch_bad(st, i);
}

struct GradPtrs {
  const float* p[kMaxReplicas];
};

__global__ void grad_mean_kernel(GradPtrs gp, int members, uint64_t n, float* __restrict__ out) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const float inv = (float)members;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    float acc = 0.0f;
    for (int a = 0; a < members; ++a) acc += gp.p[a][i];  // member order
    out[i] = acc / inv;
  }
}

__global__ void unpack_values_kernel(const uint8_t* __restrict__ vals, uint64_t n, int dtype,
                                     float* __restrict__ out) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    out[i] = load_wire_value(vals, i, dtype);
}

__global__ void striding_iota_kernel(uint32_t* __restrict__ out, uint64_t offset, uint64_t period,
                                     uint64_t count) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < count; j += stride)
    out[j] = (uint32_t)(offset + j * period);
}

}  // namespace

void launch_striding_iota(uint32_t* out, uint64_t offset, uint64_t period, uint64_t count,
                          cudaStream_t stream) {
  count_launches(1);
  if (count) striding_iota_kernel<<<grid_for(count), kBlock, 0, stream>>>(out, offset, period, count);
}

void launch_sparse_encode(const SparseSel& sel, bool sgd, const float* g, const float* m_in,
                          float* m_out, float beta, float* local_q, float* m_accum,
                          uint8_t* vals, int dtype, bool sign_mode, DevStatus* st,
                          cudaStream_t stream) {
  count_launches(1);
  sparse_encode_kernel<<<grid_for(sel.len), kBlock, 0, stream>>>(
      sel, sgd, g, m_in, m_out, beta, local_q, m_accum, vals, dtype, sign_mode, st);
}

void launch_sparse_merge_apply(const SparseSel& sel, const Bodies& in, int dtype, int mode,
                               const float* g, const float* p_in, float* p_out,
                               const float* ea_in, float* ea_out, const float* es_in,
                               float* es_out, float* q_out, SgdScalars sgd, AdamScalars adam,
                               DevStatus* st, cudaStream_t stream) {
  count_launches(1);
  const unsigned grid = grid_for(sel.len);
  if (mode == kMergeSgd)
    sparse_merge_kernel<kMergeSgd><<<grid, kBlock, 0, stream>>>(
        sel, in, dtype, g, p_in, p_out, ea_in, ea_out, es_in, es_out, q_out, sgd, adam, st);
  else if (mode == kMergeAdam)
    sparse_merge_kernel<kMergeAdam><<<grid, kBlock, 0, stream>>>(
        sel, in, dtype, g, p_in, p_out, ea_in, ea_out, es_in, es_out, q_out, sgd, adam, st);
  else
    sparse_merge_kernel<kMergeOnly><<<grid, kBlock, 0, stream>>>(
        sel, in, dtype, g, p_in, p_out, ea_in, ea_out, es_in, es_out, q_out, sgd, adam, st);
}

void launch_sgd_apply(float* p, const float* q, uint64_t n, float lr, const DevStatus* st,
                      cudaStream_t stream) {
  count_launches(1);
  sgd_apply_kernel<<<grid_for(n), kBlock, 0, stream>>>(p, q, n, lr, st);
}

void launch_adamw_apply(float* p, float* ea, float* es, const float* g, const float* lq,
                        const float* merged, uint64_t n, AdamScalars a, const DevStatus* st,
                        cudaStream_t stream) {
  count_launches(1);
  adamw_apply_kernel<<<grid_for(n), kBlock, 0, stream>>>(p, ea, es, g, lq, merged, n, a, st);
}

void launch_baseline_sgd(float* p, float* m, const float* g, uint64_t n, float beta, float lr,
                         DevStatus* st, cudaStream_t stream) {
  count_launches(2);
  check_finite_kernel<<<grid_for(n), kBlock, 0, stream>>>(g, n, st);
  baseline_sgd_kernel<<<grid_for(n), kBlock, 0, stream>>>(p, m, g, n, beta, lr, st);
}

void launch_check_finite(const float* g, uint64_t n, DevStatus* st, cudaStream_t stream) {
  count_launches(1);
  check_finite_kernel<<<grid_for(n), kBlock, 0, stream>>>(g, n, st);
}

void launch_grad_mean(const float* const* grads, int members, uint64_t n, float* out,
                      cudaStream_t stream) {
  count_launches(1);
  GradPtrs gp{};
  for (int a = 0; a < members && a < kMaxReplicas; ++a) gp.p[a] = grads[a];
  grad_mean_kernel<<<grid_for(n), kBlock, 0, stream>>>(gp, members, n, out);
}

void launch_unpack_values(const uint8_t* vals, uint64_t n, int dtype, float* out,
                          cudaStream_t stream) {
  count_launches(1);
  unpack_values_kernel<<<grid_for(n), kBlock, 0, stream>>>(vals, n, dtype, out);
}

}  // namespace dmb
