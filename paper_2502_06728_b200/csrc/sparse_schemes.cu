// sparse_schemes.cu -- Full / DiLoCo / Striding / Random encode + merge + apply,
// and the standalone elementwise optimizer kernels.  All HBM-bound: grid-stride
// loops sized to a multiple of the SM count.  The scheme kernels are specialised per
// scheme and move four consecutive elements per thread-iteration with 128-bit loads and
// stores of the dense vectors (g, m, p, moments, local_q; the Full / DiLoCo payload too);
// the Striding slot comes from a residue carried from iteration to iteration (no 64-bit
// division per element), the Random slot from the bitmap word and its prefix rank.  A
// misaligned or short vector takes the scalar kernels.
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
      float p = p_in[i] - A.lr * adam_ratio(ea, es, A);
      if (A.lr_wd != 0.0f) p -= A.lr_wd * p;
      ea_out[i] = ea;
      es_out[i] = es;
      p_out[i] = p;
    }
  }
}

// ---- vectorised scheme kernels: four consecutive elements i0 .. i0+3 per iteration ----
enum : int { kSchNone = 0, kSchDense = 1, kSchStride = 2, kSchRandom = 3 };

// Striding position of element i0 (i0 >= offset): k = i0 - offset = q * period + r
struct StrideState {
  uint64_t q, r;
};
__device__ __forceinline__ StrideState stride_at(const SparseSel& s, uint64_t i0) {
  if (i0 < s.offset) return {0, 0};
  const uint64_t k = i0 - s.offset;
  return {k / s.period, k % s.period};
}
// advance by `adv` elements, given adv = aq * period + ar (ar < period)
__device__ __forceinline__ void stride_adv(StrideState& st, uint64_t aq, uint64_t ar, uint64_t period) {
  st.q += aq;
  st.r += ar;
  if (st.r >= period) {
    st.r -= period;
    ++st.q;
  }
}

// selection mask (bit j: element i0 + j transmitted) and the slot of the first selected one;
// the selected elements of a quad occupy consecutive slots (Random, Striding with period 1)
// or one slot each (Striding), so slot(j) = base + rank of j among the selected
template <int SCH>
__device__ __forceinline__ uint32_t quad_sel(const SparseSel& s, uint64_t i0, const StrideState& st,
                                             uint64_t (&slot)[4]) {
  uint32_t m = 0;
  if (SCH == kSchDense) {
#pragma unroll
    for (int j = 0; j < 4; ++j) slot[j] = i0 + j;
    return i0 + 4 <= s.len ? 0xFu : (1u << (s.len - i0)) - 1u;
  }
  if (SCH == kSchRandom) {
    const uint32_t w = s.bitmap[i0 >> 5];
    const uint32_t sh = (uint32_t)(i0 & 31);
    m = (w >> sh) & 0xFu;
    uint64_t base = s.rank[i0 >> 5] + __popc(w & ((1u << sh) - 1u));
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      slot[j] = base;
      base += (m >> j) & 1u;
    }
    return m;
  }
  if (SCH == kSchStride) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint64_t i = i0 + j;
      if (i < s.offset || i >= s.len) continue;
      // element i0 + j: residue r + j - (i0 < offset adjustments are excluded above)
      uint64_t r = st.r + (i0 >= s.offset ? (uint64_t)j : i - s.offset), q = st.q;
      if (i0 < s.offset) {
        r = i - s.offset;
        q = 0;
      }
      while (r >= s.period) {
        r -= s.period;
        ++q;
      }
      if (r == 0) {
        m |= 1u << j;
        slot[j] = q;
      }
    }
    return m;
  }
  return 0u;
}

template <int SCH>
__global__ void __launch_bounds__(kBlock) sparse_encode_v4(SparseSel sel, bool sgd, const float* __restrict__ g,
                                                           const float* __restrict__ m_in, float* __restrict__ m_out,
                                                           float beta, float* __restrict__ local_q,
                                                           float* __restrict__ m_accum, uint8_t* __restrict__ vals,
                                                           int dtype, bool sign_mode, DevStatus* st) {
  const uint64_t nq = (sel.len + 3) / 4;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  uint64_t qd = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  StrideState ss{0, 0};
  uint64_t aq = 0, ar = 0;
  bool ss_valid = false;  // the carried residue is exact once the quad starts at or after offset
  if (SCH == kSchStride) {
    ss = stride_at(sel, 4 * qd);
    ss_valid = 4 * qd >= sel.offset;
    aq = (4 * stride) / sel.period;
    ar = (4 * stride) % sel.period;
  }
  for (; qd < nq; qd += stride) {
    const uint64_t i0 = 4 * qd;
    const bool full = i0 + 4 <= sel.len;
    float x[4], gi[4];
    if (full) {
      const float4 gv = *reinterpret_cast<const float4*>(g + i0);
      gi[0] = gv.x, gi[1] = gv.y, gi[2] = gv.z, gi[3] = gv.w;
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) gi[j] = i0 + j < sel.len ? g[i0 + j] : 0.0f;
    }
    float mi[4] = {0.f, 0.f, 0.f, 0.f};
    if (sgd) {
      if (full) {
        const float4 mv = *reinterpret_cast<const float4*>(m_in + i0);
        mi[0] = mv.x, mi[1] = mv.y, mi[2] = mv.z, mi[3] = mv.w;
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) mi[j] = i0 + j < sel.len ? m_in[i0 + j] : 0.0f;
      }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (!isfinite(gi[j]) && i0 + j < sel.len) latch_bad(st, i0 + j);
      x[j] = sgd ? __fadd_rn(__fmul_rn(beta, mi[j]), gi[j]) : gi[j];  // optim.cpp:27
    }
    uint64_t slot[4];
    const uint32_t on = quad_sel<SCH>(sel, i0, ss, slot);
    if (vals && on) {
      if (SCH == kSchDense && full && dtype == DMB_FP32 && !sign_mode) {
        *reinterpret_cast<float4*>(reinterpret_cast<float*>(vals) + i0) = make_float4(x[0], x[1], x[2], x[3]);
      } else if (SCH == kSchDense && dtype == DMB_TERNARY) {
        uint32_t b = 0;  // the quad's four 2-bit codes are one byte of the body (LSB first)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float c = sign_of(x[j]);
          if ((on >> j) & 1u) b |= (c > 0.0f ? 1u : (c < 0.0f ? 2u : 0u)) << (2 * j);
        }
        vals[i0 >> 2] = (uint8_t)b;
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if ((on >> j) & 1u) store_wire_value(vals, slot[j], condition_f32(x[j], dtype, sign_mode), dtype);
      }
    }
    float lq[4], mo[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const bool sj = (on >> j) & 1u;
      lq[j] = sj ? x[j] : 0.0f;
      mo[j] = sj ? x[j] - x[j] : x[j];  // optim.cpp:35-37 with local_q = x or 0
    }
    if (full) {
      if (m_accum) *reinterpret_cast<float4*>(m_accum + i0) = make_float4(x[0], x[1], x[2], x[3]);
      if (local_q) *reinterpret_cast<float4*>(local_q + i0) = make_float4(lq[0], lq[1], lq[2], lq[3]);
      if (sgd) *reinterpret_cast<float4*>(m_out + i0) = make_float4(mo[0], mo[1], mo[2], mo[3]);
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (i0 + j < sel.len) {
          if (m_accum) m_accum[i0 + j] = x[j];
          if (local_q) local_q[i0 + j] = lq[j];
          if (sgd) m_out[i0 + j] = mo[j];
        }
    }
    if (SCH == kSchStride) {
      if (ss_valid) {
        stride_adv(ss, aq, ar, sel.period);
      } else {
        ss = stride_at(sel, 4 * (qd + stride));
        ss_valid = 4 * (qd + stride) >= sel.offset;
      }
    }
  }
}

__device__ __forceinline__ float4 ld4(const float* p) { return *reinterpret_cast<const float4*>(p); }
__device__ __forceinline__ void st4(float* p, const float (&v)[4]) {
  *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
}

template <int SCH, int MODE>
__global__ void __launch_bounds__(kBlock) sparse_merge_v4(SparseSel sel, Bodies in, int dtype,
                                                          const float* __restrict__ g, const float* __restrict__ p_in,
                                                          float* __restrict__ p_out, const float* __restrict__ ea_in,
                                                          float* __restrict__ ea_out,
                                                          const float* __restrict__ es_in,
                                                          float* __restrict__ es_out, float* __restrict__ q_out,
                                                          SgdScalars sgd, AdamScalars A, DevStatus* st) {
  if (step_failed(st)) return;
  const uint64_t nq = (sel.len + 3) / 4;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const float R = (float)in.R;
  // the merged value of a ternary member sum x is x / R: the 2R + 1 possible quotients, IEEE
  // divided once per CTA (the division per element cost more than the memory traffic)
  __shared__ float qtab[2 * 120 + 1];
  // x / R for a power-of-two R is x * (1 / R) exactly: a multiply instead of the IEEE division
  const bool pow2 = (in.R & (in.R - 1)) == 0;
  const float invR = 1.0f / R;
  auto div_r = [&](float x) { return pow2 ? x * invR : x / R; };
  const bool tern = SCH == kSchDense && dtype == DMB_TERNARY && in.R <= 120;
  if (tern) {
    for (int x = threadIdx.x; x <= 2 * in.R; x += blockDim.x) qtab[x] = (float)(x - in.R) / R;
    __syncthreads();
  }
  uint64_t qd = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  StrideState ss{0, 0};
  uint64_t aq = 0, ar = 0;
  bool ss_valid = false;  // the carried residue is exact once the quad starts at or after offset
  if (SCH == kSchStride) {
    ss = stride_at(sel, 4 * qd);
    ss_valid = 4 * qd >= sel.offset;
    aq = (4 * stride) / sel.period;
    ar = (4 * stride) % sel.period;
  }
  for (; qd < nq; qd += stride) {
    const uint64_t i0 = 4 * qd;
    const bool full = i0 + 4 <= sel.len;
    uint64_t slot[4];
    const uint32_t on = quad_sel<SCH>(sel, i0, ss, slot);
    float q[4] = {0.f, 0.f, 0.f, 0.f};
    if (SCH == kSchDense && full && dtype == DMB_FP32) {
      float acc[4] = {0.f, 0.f, 0.f, 0.f};  // member order (replicate.cpp:264-265)
      for (int r0 = 0; r0 < in.R; r0 += 4) {  // four members' loads in flight, then added in order
        float4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          v[u] = r0 + u < in.R ? ld4(reinterpret_cast<const float*>(in.body[r0 + u]) + i0) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (r0 + u < in.R) acc[0] += v[u].x, acc[1] += v[u].y, acc[2] += v[u].z, acc[3] += v[u].w;
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) q[j] = div_r(acc[j]);
    } else if (tern && full) {
      // the quad's four 2-bit codes are one byte of every body; a member's values are -1 / 0 / +1,
      // so their member-order FP32 sum is an exact integer: count it in byte lanes (value + 1 =
      // (code & 1) + (~code >> 1 & 1) per field: 1 -> 2, 2 -> 0, 0 and 3 -> 1), one load per member
      // (members in groups of eight whose loads are all issued before any is used: one memory
      // latency per group, not per member)
      uint32_t cnt = 0;
      for (int r0 = 0; r0 < in.R; r0 += 8) {
        uint32_t bb[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) bb[u] = r0 + u < in.R ? (uint32_t)__ldg(in.body[r0 + u] + (i0 >> 2)) : 0x55u;
#pragma unroll
        for (int u = 0; u < 8; ++u) {  // the padding code 0x55 (+1 x 4) is taken back below
          const uint32_t b = bb[u];
          const uint32_t t = (b & 0x55u) + (~(b >> 1) & 0x55u);
          cnt += (t & 3u) | ((t & 0xCu) << 6) | ((t & 0x30u) << 12) | ((t & 0xC0u) << 18);
        }
      }
      const int pad = (8 - in.R % 8) % 8;  // padding members counted value + 1 = 2 each
      cnt -= (uint32_t)(2 * pad) * 0x01010101u;  // byte j: x + R for the sum x of element j
#pragma unroll
      for (int j = 0; j < 4; ++j) q[j] = qtab[(cnt >> (8 * j)) & 0xffu];
    } else if (on) {
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if ((on >> j) & 1u) {
          float acc = 0.0f;  // member order (replicate.cpp:264-265, :277-279)
          for (int r = 0; r < in.R; ++r) acc += load_wire_value(in.body[r], slot[j], dtype);
          q[j] = div_r(acc);
        }
    }
    if (full) {
      if (q_out) st4(q_out + i0, q);
      if (MODE == kMergeSgd) {
        const float4 pv = ld4(p_in + i0);
        const float pr[4] = {pv.x - sgd.lr * q[0], pv.y - sgd.lr * q[1], pv.z - sgd.lr * q[2], pv.w - sgd.lr * q[3]};
        st4(p_out + i0, pr);
      } else if (MODE == kMergeAdam) {
        const float4 gv = ld4(g + i0), pv = ld4(p_in + i0), ev = ld4(ea_in + i0), sv = ld4(es_in + i0);
        const float gi[4] = {gv.x, gv.y, gv.z, gv.w}, pi[4] = {pv.x, pv.y, pv.z, pv.w};
        const float ei[4] = {ev.x, ev.y, ev.z, ev.w}, si[4] = {sv.x, sv.y, sv.z, sv.w};
        float po[4], eo[4], so[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          // g' = g - local_q + merged with local_q = g on selected slots, else 0
          const float gp = ((on >> j) & 1u) ? (gi[j] - gi[j]) + q[j] : (gi[j] - 0.0f) + q[j];
          eo[j] = A.beta1 * ei[j] + A.one_minus_beta1 * gp;
          so[j] = A.beta2 * si[j] + A.one_minus_beta2 * gp * gp;
          float pn = pi[j] - A.lr * adam_ratio(eo[j], so[j], A);
          if (A.lr_wd != 0.0f) pn -= A.lr_wd * pn;
          po[j] = pn;
        }
        st4(p_out + i0, po);
        st4(ea_out + i0, eo);
        st4(es_out + i0, so);
      }
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint64_t i = i0 + j;
        if (i >= sel.len) break;
        if (q_out) q_out[i] = q[j];
        if (MODE == kMergeSgd) {
          p_out[i] = p_in[i] - sgd.lr * q[j];
        } else if (MODE == kMergeAdam) {
          const float gi = g[i];
          const float gp = ((on >> j) & 1u) ? (gi - gi) + q[j] : (gi - 0.0f) + q[j];
          const float ea = A.beta1 * ea_in[i] + A.one_minus_beta1 * gp;
          const float es = A.beta2 * es_in[i] + A.one_minus_beta2 * gp * gp;
          float pn = p_in[i] - A.lr * adam_ratio(ea, es, A);
          if (A.lr_wd != 0.0f) pn -= A.lr_wd * pn;
          ea_out[i] = ea;
          es_out[i] = es;
          p_out[i] = pn;
        }
      }
    }
    if (SCH == kSchStride) {
      if (ss_valid) {
        stride_adv(ss, aq, ar, sel.period);
      } else {
        ss = stride_at(sel, 4 * (qd + stride));
        ss_valid = 4 * (qd + stride) >= sel.offset;
      }
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
    float pv = p[i] - A.lr * adam_ratio(ea, es, A);
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

// grad_reduce_scatter's member-order mean (vec.cpp:18-26, cluster.cpp:63-91) with a CTA budget: a
// persistent grid of `ctas` CTAs that can run beside a step kernel leaving those SMs free (the
// cluster's reduce-scatter of bucket b+1 under the prepare of bucket b).  Few CTAs must still move
// HBM-rate bytes, so the latency is hidden by loads in flight, not by occupancy: every thread
// issues kPullUnroll 16-byte loads of every member (the member count a template parameter for
// 2-4) before summing them -- from 0, members in order, then divided, as mean_of does.
constexpr int kPullThreads = 512;
constexpr int kPullUnroll = 8;

template <int M>  // members; 0: run-time count
__global__ void __launch_bounds__(kPullThreads) grad_mean_pull_kernel(GradPtrs gp, int members, uint64_t n4,
                                                                      float4* __restrict__ out) {
  const int nm = M > 0 ? M : members;
  const float inv = (float)nm;
  const uint64_t stride = (uint64_t)gridDim.x * kPullThreads;
  for (uint64_t i0 = (uint64_t)blockIdx.x * kPullThreads + threadIdx.x; i0 < n4; i0 += stride * kPullUnroll) {
    float4 acc[kPullUnroll];
#pragma unroll
    for (int u = 0; u < kPullUnroll; ++u) acc[u] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (M > 0) {
      float4 v[M > 0 ? M : 1][kPullUnroll];
#pragma unroll
      for (int a = 0; a < (M > 0 ? M : 1); ++a) {
        const float4* src = reinterpret_cast<const float4*>(gp.p[a]);
#pragma unroll
        for (int u = 0; u < kPullUnroll; ++u) {
          const uint64_t i = i0 + u * stride;
          v[a][u] = i < n4 ? __ldcg(src + i) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
#pragma unroll
      for (int a = 0; a < (M > 0 ? M : 1); ++a)
#pragma unroll
        for (int u = 0; u < kPullUnroll; ++u) {
          acc[u].x += v[a][u].x;
          acc[u].y += v[a][u].y;
          acc[u].z += v[a][u].z;
          acc[u].w += v[a][u].w;
        }
    } else {
      for (int a = 0; a < nm; ++a) {
        const float4* src = reinterpret_cast<const float4*>(gp.p[a]);
        float4 v[kPullUnroll];
#pragma unroll
        for (int u = 0; u < kPullUnroll; ++u) {
          const uint64_t i = i0 + u * stride;
          v[u] = i < n4 ? __ldcg(src + i) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int u = 0; u < kPullUnroll; ++u) {
          acc[u].x += v[u].x;
          acc[u].y += v[u].y;
          acc[u].z += v[u].z;
          acc[u].w += v[u].w;
        }
      }
    }
#pragma unroll
    for (int u = 0; u < kPullUnroll; ++u) {
      const uint64_t i = i0 + u * stride;
      if (i < n4) out[i] = make_float4(acc[u].x / inv, acc[u].y / inv, acc[u].z / inv, acc[u].w / inv);
    }
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
  auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; };
  const bool v4 = al(g) && (!sgd || (al(m_in) && al(m_out))) && al(local_q) && al(m_accum) &&
                  (sel.scheme != DMB_FULL && sel.scheme != DMB_DILOCO ? true : al(vals));
  const unsigned grid = grid_for((sel.len + 3) / 4);
  if (v4) {
    switch (sel.scheme) {
      case 0: sparse_encode_v4<kSchNone><<<grid, kBlock, 0, stream>>>(sel, sgd, g, m_in, m_out, beta, local_q, m_accum, vals, dtype, sign_mode, st); return;
      case DMB_FULL:
      case DMB_DILOCO: sparse_encode_v4<kSchDense><<<grid, kBlock, 0, stream>>>(sel, sgd, g, m_in, m_out, beta, local_q, m_accum, vals, dtype, sign_mode, st); return;
      case DMB_STRIDING: sparse_encode_v4<kSchStride><<<grid, kBlock, 0, stream>>>(sel, sgd, g, m_in, m_out, beta, local_q, m_accum, vals, dtype, sign_mode, st); return;
      default: sparse_encode_v4<kSchRandom><<<grid, kBlock, 0, stream>>>(sel, sgd, g, m_in, m_out, beta, local_q, m_accum, vals, dtype, sign_mode, st); return;
    }
  }
  sparse_encode_kernel<<<grid_for(sel.len), kBlock, 0, stream>>>(
      sel, sgd, g, m_in, m_out, beta, local_q, m_accum, vals, dtype, sign_mode, st);
}

void launch_sparse_merge_apply(const SparseSel& sel, const Bodies& in, int dtype, int mode,
                               const float* g, const float* p_in, float* p_out,
                               const float* ea_in, float* ea_out, const float* es_in,
                               float* es_out, float* q_out, SgdScalars sgd, AdamScalars adam,
                               DevStatus* st, cudaStream_t stream) {
  count_launches(1);
  auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; };
  bool v4 = al(g) && al(p_in) && al(p_out) && al(ea_in) && al(ea_out) && al(es_in) && al(es_out) && al(q_out);
  for (int r = 0; r < in.R && v4; ++r) v4 = al(in.body[r]) || (sel.scheme != DMB_FULL && sel.scheme != DMB_DILOCO);
  if (v4) {
    const unsigned g4 = grid_for((sel.len + 3) / 4);
#define DMB_MERGE_V4(SCH)                                                                                   \
  do {                                                                                                     \
    if (mode == kMergeSgd)                                                                                 \
      sparse_merge_v4<SCH, kMergeSgd><<<g4, kBlock, 0, stream>>>(sel, in, dtype, g, p_in, p_out, ea_in,    \
                                                                 ea_out, es_in, es_out, q_out, sgd, adam, st); \
    else if (mode == kMergeAdam)                                                                           \
      sparse_merge_v4<SCH, kMergeAdam><<<g4, kBlock, 0, stream>>>(sel, in, dtype, g, p_in, p_out, ea_in,   \
                                                                  ea_out, es_in, es_out, q_out, sgd, adam, st); \
    else                                                                                                   \
      sparse_merge_v4<SCH, kMergeOnly><<<g4, kBlock, 0, stream>>>(sel, in, dtype, g, p_in, p_out, ea_in,   \
                                                                  ea_out, es_in, es_out, q_out, sgd, adam, st); \
  } while (0)
    switch (sel.scheme) {
      case DMB_FULL:
      case DMB_DILOCO: DMB_MERGE_V4(kSchDense); return;
      case DMB_STRIDING: DMB_MERGE_V4(kSchStride); return;
      case DMB_RANDOM: DMB_MERGE_V4(kSchRandom); return;
      default: break;
    }
#undef DMB_MERGE_V4
  }
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

void launch_grad_mean_pull(const float* const* grads, int members, uint64_t n, float* out, int ctas,
                           cudaStream_t stream) {
  GradPtrs gp{};
  bool al = (reinterpret_cast<uintptr_t>(out) & 15u) == 0;
  for (int a = 0; a < members && a < kMaxReplicas; ++a) {
    gp.p[a] = grads[a];
    al = al && (reinterpret_cast<uintptr_t>(grads[a]) & 15u) == 0;
  }
  const uint64_t n4 = al ? n / 4 : 0;
  if (n4) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const uint64_t want = (n4 + (uint64_t)kPullThreads * kPullUnroll - 1) / ((uint64_t)kPullThreads * kPullUnroll);
    const uint64_t cap = (uint64_t)(ctas > 0 ? ctas : sms);
    count_launches(1);
    const unsigned grid = (unsigned)(want < cap ? want : cap);
    float4* o4 = reinterpret_cast<float4*>(out);
    switch (members) {
      case 2: grad_mean_pull_kernel<2><<<grid, kPullThreads, 0, stream>>>(gp, members, n4, o4); break;
      case 3: grad_mean_pull_kernel<3><<<grid, kPullThreads, 0, stream>>>(gp, members, n4, o4); break;
      case 4: grad_mean_pull_kernel<4><<<grid, kPullThreads, 0, stream>>>(gp, members, n4, o4); break;
      default: grad_mean_pull_kernel<0><<<grid, kPullThreads, 0, stream>>>(gp, members, n4, o4);
    }
  }
  if (n4 * 4 < n) {  // the tail, or every element of a misaligned vector
    GradPtrs gt{};
    for (int a = 0; a < members && a < kMaxReplicas; ++a) gt.p[a] = grads[a] + n4 * 4;
    count_launches(1);
    grad_mean_kernel<<<grid_for(n - n4 * 4), kBlock, 0, stream>>>(gt, members, n - n4 * 4, out + n4 * 4);
  }
}

void launch_unpack_values(const uint8_t* vals, uint64_t n, int dtype, float* out,
                          cudaStream_t stream) {
  count_launches(1);
  unpack_values_kernel<<<grid_for(n), kBlock, 0, stream>>>(vals, n, dtype, out);
}

}  // namespace dmb
