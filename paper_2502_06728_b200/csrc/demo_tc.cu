// demo_tc.cu -- the DeMo hot path for chunk size 64 on the 5th-generation tensor
// cores (tcgen05, sm_100a).
//
// A tile is 128 consecutive chunks of the shard (8192 parameters).  Per tile:
//   1. every thread owns one chunk (row): loads it (m = beta m + g fused, finite
//      check), splits it into TF32 hi/lo and writes both into K-major SW128 smem;
//   2. one thread issues the forward DCT  C = X B^T  as 3xTF32 tcgen05.mma
//      (Xhi Bhi + Xhi Blo + Xlo Bhi, M=128 N=64 K=64) into TMEM;
//   3. tcgen05.ld moves each row's 64 coefficients into that thread's registers:
//      TopK by MSB radix select (ties -> lower index), certification against the
//      FP64 oracle (error bound below), payload (indices + conditioned values);
//      uncertain rows are handed to the FP64 re-derivation kernel and skipped here;
//   4. the inverse DCT of what the optimizer needs (Q - local_q for AdamW; local_q
//      and Q for SGD) runs as a second 3xTF32 MMA;
//   5. the epilogue applies m <- m_acc - local_q, p <- p - lr Q or the AdamW update.
// Two independent 4-warp groups per CTA work on different tiles and share the
// basis tables, so one group's memory phase overlaps the other's compute.
//
// Reference: transform.cpp:56-73 (DCT), :127-147 (TopK, sparse inverse),
// replicate.cpp:137-144 + :282-309 (conditioning, merge), optim.cpp:18-74.
//
// Certification bound: |c~_j - c_j| <= kEpsScale * ||x||_1, derived with the per-MMA model
// of demo_tc_adam.cu (at kEpsW / kEpsL there): one tcgen05.mma kind::tf32 step (K = 8) takes exact
// products, aligns every term to the largest exponent with truncation and truncates the sum
// once -> error <= 9 * 2^-23 (|acc| + sum |terms|).  With S = sum_i |x_i||B_ji| <=
// sqrt(2/s) ||x||_1 and RNA TF32 splits (|x - hi| <= 2^-11 |x|, |x - hi - lo| <= 2^-22 |x|,
// the same for B), in the issue order of issue_3x:
//   16 cross-term steps first (acc + terms <= 2 * 2^-11 (1 + 2^-11) S): 16 * 9 * 2^-23 * 2^-10 S
//                                                                       = 1.7e-8 S
//   8 hi*hi steps last (acc + terms <= (1 + 2^-9) S):  8 * 9 * 2^-23 * (1 + 2^-9) S = 8.60e-6 S
//   split residuals: x (2^-22), B (2^-22), the dropped lo*lo (2^-22)      = 7.2e-7 S
//   oracle's own FP64 rounding: 64 * 2^-53 S                               ~ 0
// total 9.34e-6 S; the radius used, 2^-16 * 1.01 = 1.54e-5 S, covers it with a 1.65x margin.
#include <cfloat>

#include "dmb_internal.cuh"
#include "tc_ptx.cuh"

namespace dmb {
namespace {

using namespace ptx;

constexpr int S = 64;
constexpr int TM = 128;
constexpr int GROUPS = 2;
constexpr int THREADS = 128 * GROUPS;
constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(S >> 3) << 17) |
                           ((uint32_t)(TM >> 4) << 24);
constexpr uint32_t B_BYTES = S * 128 * 2;   // 64 rows x 2 k-blocks x 128 B
constexpr uint32_t A_BYTES = TM * 128 * 2;  // 128 rows x 2 k-blocks x 128 B
constexpr uint32_t OFF_BHI = 0, OFF_BLO = B_BYTES, OFF_BTHI = 2 * B_BYTES, OFF_BTLO = 3 * B_BYTES;
constexpr uint32_t OFF_A = 4 * B_BYTES;
constexpr uint32_t OFF_BAR = OFF_A + GROUPS * 2 * A_BYTES;
constexpr uint32_t SMEM_BYTES = OFF_BAR + 64 + 1024;
constexpr uint32_t TMEM_COLS = 512;  // per group: D1 | D2 | D3 at +0 / +64 / +128, group stride 256
constexpr float kEpsScale = 1.52587890625e-05f * 0.1767766952966369f * 1.01f;  // 2^-16 sqrt(2/64), see above

// byte offset of the 16-byte chunk q (cols 4q..4q+3) of row r in a K-major SW128 tile
__device__ __forceinline__ uint32_t sw_off(int r, int q, uint32_t rows) {
  return (uint32_t)(q >> 3) * rows * 128u + (uint32_t)r * 128u + ((uint32_t)((q & 7) ^ (r & 7)) << 4);
}

// Row r of an A operand: value(j) for j = 0..63 as TF32 hi/lo (RNA splits), or as
// exact hi with lo = 0 when every value is TF32-exact (signs, fp16-rounded values).
template <typename F>
__device__ __forceinline__ void store_row(uint8_t* hi_base, uint8_t* lo_base, int r, bool exact, F value) {
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    float v[4], h[4], l[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      v[e] = value(4 * q + e);
      h[e] = exact ? v[e] : tf32_rna(v[e]);
      l[e] = exact ? 0.0f : tf32_rna(v[e] - h[e]);
    }
    const uint32_t off = sw_off(r, q, TM);
    *reinterpret_cast<float4*>(hi_base + off) = make_float4(h[0], h[1], h[2], h[3]);
    *reinterpret_cast<float4*>(lo_base + off) = make_float4(l[0], l[1], l[2], l[3]);
  }
}

// D = Ahi Bhi + Ahi Blo + Alo Bhi over K = 64 (8 MMAs of K = 8 per product).  The 16 small
// cross terms (|term| <= 2^-11 |x||B| each) accumulate first and the 8 hi*hi steps last, so
// the accumulator is small while the small terms are added: kEpsScale assumes this order.
__device__ __forceinline__ void issue_3x(uint32_t d, uint32_t ahi, uint32_t alo, uint32_t bhi, uint32_t blo,
                                         bool lo_a) {
  auto ao = [](int k) { return (uint32_t)(k >> 2) * (TM * 128u) + (uint32_t)(k & 3) * 32u; };
  auto bo = [](int k) { return (uint32_t)(k >> 2) * (S * 128u) + (uint32_t)(k & 3) * 32u; };
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    mma_tf32(d, desc_sw128(ahi + ao(k)), desc_sw128(blo + bo(k)), IDESC, k > 0 ? 1u : 0u);
    if (lo_a) mma_tf32(d, desc_sw128(alo + ao(k)), desc_sw128(bhi + bo(k)), IDESC, 1u);
  }
#pragma unroll
  for (int k = 0; k < 8; ++k) mma_tf32(d, desc_sw128(ahi + ao(k)), desc_sw128(bhi + bo(k)), IDESC, 1u);
}

__device__ __forceinline__ void load_tmem_row(uint32_t taddr, float (&v)[64]) {
  tmem_ld16(taddr + 0, v + 0);
  tmem_ld16(taddr + 16, v + 16);
  tmem_ld16(taddr + 32, v + 32);
  tmem_ld16(taddr + 48, v + 48);
  tmem_ld_wait();
}

// TopK over 64 register-resident |c| keys: MSB radix select with early exit.
// Returns the selection mask (bit j = frequency j), ties toward the lower index.
__device__ __forceinline__ uint64_t topk64(const float (&c)[64], int k) {
  uint32_t T = 0;
  bool exact = false;
#pragma unroll 1
  for (int b = 30; b >= 0; --b) {
    const uint32_t cand = T | (1u << b);
    int cnt = 0;
#pragma unroll
    for (int j = 0; j < 64; ++j) cnt += __float_as_uint(fabsf(c[j])) >= cand ? 1 : 0;
    if (cnt >= k) {
      T = cand;
      if (cnt == k) {
        exact = true;
        break;
      }
    }
  }
  uint64_t sel = 0;
  if (exact) {
#pragma unroll
    for (int j = 0; j < 64; ++j)
      if (__float_as_uint(fabsf(c[j])) >= T) sel |= 1ull << j;
    return sel;
  }
  int gt = 0;
#pragma unroll
  for (int j = 0; j < 64; ++j) gt += __float_as_uint(fabsf(c[j])) > T ? 1 : 0;
  int need = k - gt;
#pragma unroll
  for (int j = 0; j < 64; ++j) {
    const uint32_t key = __float_as_uint(fabsf(c[j]));
    const bool take = key > T || (key == T && need > 0);
    if (key == T && need > 0) --need;
    if (take) sel |= 1ull << j;
  }
  return sel;
}

template <ChunkMode MODE>
__global__ void __launch_bounds__(THREADS, 1) demo_tc_kernel(const ChunkArgs a) {
  constexpr bool kSgd = MODE == ChunkMode::EncodeSgd || MODE == ChunkMode::StepSgd;
  constexpr bool kStep = MODE == ChunkMode::StepSgd || MODE == ChunkMode::StepAdam;
  constexpr bool kAdamStep = MODE == ChunkMode::StepAdam;

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + OFF_BAR);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + OFF_BAR + 32);

  const int tid = threadIdx.x;
  const int grp = tid >> 7;
  const int t = tid & 127;
  const int warp = tid >> 5;

  if (kStep && step_failed(a.status)) return;

  // ---- one-time setup: basis tables -> swizzled smem, barriers, TMEM ----
  {
    const float* src[4] = {a.basis.Bhi, a.basis.Blo, a.basis.BThi, a.basis.BTlo};
    for (int m = 0; m < 4; ++m) {
      uint8_t* dst = smem + m * B_BYTES;
      for (int u = tid; u < S * 16; u += THREADS) {
        const int r = u >> 4, q = u & 15;
        *reinterpret_cast<float4*>(dst + sw_off(r, q, S)) =
            *reinterpret_cast<const float4*>(src[m] + r * S + 4 * q);
      }
    }
  }
  if (tid == 0) {
    for (int g = 0; g < GROUPS; ++g) mbar_init(&bars[g], 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(tmem_slot, TMEM_COLS);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const uint32_t s_base = smem_u32(smem);
  const uint32_t bhi = s_base + OFF_BHI, blo = s_base + OFF_BLO;
  const uint32_t bthi = s_base + OFF_BTHI, btlo = s_base + OFF_BTLO;
  uint8_t* a_hi = smem + OFF_A + grp * 2 * A_BYTES;
  uint8_t* a_lo = a_hi + A_BYTES;
  const uint32_t ahi = smem_u32(a_hi), alo = smem_u32(a_lo);
  const uint32_t tm = tmem_base + (uint32_t)grp * 256u;            // this group's columns
  const uint32_t tm_row = tm + ((uint32_t)((warp & 3) * 32) << 16);  // this warp's lane quadrant
  uint64_t* bar = &bars[grp];
  uint32_t phase = 0;

  const uint64_t len = a.geo.len;
  const uint64_t nchunks = a.geo.nchunks;
  const uint64_t ntiles = (nchunks + TM - 1) / TM;
  const int k = a.geo.k;
  const int dtype = a.geo.dtype;
  const bool sign_mode = a.geo.sign_mode;
  const bool need_signs = sign_mode || dtype == DMB_TERNARY;
  const uint64_t nvals = nchunks * (uint64_t)k;
  const bool full_band = k == S;

  for (uint64_t tile = (uint64_t)blockIdx.x * GROUPS + grp; tile < ntiles; tile += (uint64_t)gridDim.x * GROUPS) {
    const uint64_t row = tile * TM + t;
    const bool row_ok = row < nchunks;
    const uint64_t base = row * S;
    const bool whole = row_ok && base + S <= len;

    // ---- 1. load the chunk, fuse the momentum accumulate, split into TF32 hi/lo ----
    float x[64];
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      float4 gv = make_float4(0.f, 0.f, 0.f, 0.f), mv = make_float4(0.f, 0.f, 0.f, 0.f);
      if (whole) {
        gv = __ldcs(reinterpret_cast<const float4*>(a.g + base) + q);
        if (kSgd) mv = __ldcs(reinterpret_cast<const float4*>(a.m_in + base) + q);
      } else if (row_ok) {
        float* gp = &gv.x;
        float* mp = &mv.x;
        for (int e = 0; e < 4; ++e) {
          const uint64_t i = base + 4 * q + e;
          if (i < len) {
            gp[e] = a.g[i];
            if (kSgd) mp[e] = a.m_in[i];
          }
        }
      }
      const float* gp = &gv.x;
      const float* mp = &mv.x;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        if (!isfinite(gp[e])) latch_bad(a.status, base + 4 * q + e);
        x[4 * q + e] = kSgd ? __fadd_rn(__fmul_rn(a.sgd.beta, mp[e]), gp[e]) : gp[e];  // optim.cpp:27
      }
    }
    float l1 = 0.f;
#pragma unroll
    for (int j = 0; j < 64; ++j) l1 += fabsf(x[j]);
    store_row(a_hi, a_lo, t, false, [&](int j) { return x[j]; });
    fence_proxy_async_smem();
    named_sync(1 + grp, 128);

    // ---- 2. forward DCT on the tensor cores ----
    if (t == 0) {
      tc_fence_after();
      issue_3x(tm + 0, ahi, alo, bhi, blo, true);
      mma_commit(bar);
    }
    mbar_wait(bar, phase);
    phase ^= 1;
    tc_fence_after();

    // ---- 3. TopK + certification + payload, per row ----
    float c[64];
    load_tmem_row(tm_row + 0, c);
    uint64_t sel = full_band ? ~0ull : topk64(c, k);
    bool skip = !row_ok;
    if (row_ok) {
      float kth = FLT_MAX, nxt = 0.f;
#pragma unroll
      for (int j = 0; j < 64; ++j) {
        const float m = fabsf(c[j]);
        if ((sel >> j) & 1ull) kth = fminf(kth, m);
        else nxt = fmaxf(nxt, m);
      }
      const float eps = kEpsScale * l1;
      bool uncertain = full_band ? (need_signs && !(kth > eps)) : !(kth - nxt > 2.0f * eps);
      if (isnan(l1)) uncertain = false;  // non-finite input: the step fails anyway
      if (uncertain || a.force_fp64) {
        const unsigned slot = atomicAdd(a.fb_count, 1u);
        a.fb_list[slot] = (uint32_t)row;
        skip = true;
      }
    }
    auto wire = [&](int j) -> float {  // conditioned wire value (0 where not selected)
      return ((sel >> j) & 1ull) ? condition_f32(c[j], dtype, sign_mode) : 0.0f;
    };
    if (!skip && a.body) {
      uint32_t* idx_out = reinterpret_cast<uint32_t*>(a.body) + row * (uint64_t)k;
      uint8_t* val_out = a.body + nvals * 4;
      uint64_t tpos = row * (uint64_t)k;
#pragma unroll
      for (int j = 0; j < 64; ++j) {
        if ((sel >> j) & 1ull) {
          *idx_out++ = (uint32_t)j;
          store_wire_value(val_out, tpos++, wire(j), dtype);
        }
      }
    }

    // ---- 4. inverse DCT operand(s) ----
    // StepAdam: W = wire - coef on the selection (Q - local_q in one transform);
    //           full band: W = wire (local_q == x exactly).
    // SGD / local_q: W1 = coef on the selection (local_q); StepSgd adds W2 = wire (Q).
    const bool exact_w = kAdamStep && full_band && (need_signs || dtype == DMB_FP16);
    if (kAdamStep) {
      store_row(a_hi, a_lo, t, exact_w, [&](int j) -> float {
        return full_band ? wire(j) : (((sel >> j) & 1ull) ? wire(j) - c[j] : 0.0f);
      });
    } else {
      store_row(a_hi, a_lo, t, false, [&](int j) -> float { return ((sel >> j) & 1ull) ? c[j] : 0.0f; });
    }
    const bool need_lq = !(full_band && kSgd) && (kSgd || a.local_q != nullptr || kAdamStep);
    fence_proxy_async_smem();
    tc_fence_before();
    named_sync(1 + grp, 128);
    if (need_lq) {
      if (t == 0) {
        tc_fence_after();
        issue_3x(tm + 64, ahi, alo, bthi, btlo, !exact_w);
        mma_commit(bar);
      }
      mbar_wait(bar, phase);
      phase ^= 1;
      tc_fence_after();
    }

    // ---- 5. epilogue ----
    if (kAdamStep) {
      float d[64];
      load_tmem_row(tm_row + 64, d);
      if (!skip) {
        const AdamScalars& A = a.adam;
        const bool whole_out = whole;
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          float4 pv, ev, sv;
          const uint64_t i0 = base + 4 * q;
          if (whole_out) {
            pv = *reinterpret_cast<const float4*>(a.p_in + i0);
            ev = *reinterpret_cast<const float4*>(a.ea_in + i0);
            sv = *reinterpret_cast<const float4*>(a.es_in + i0);
          } else {
            pv = ev = sv = make_float4(0.f, 0.f, 0.f, 0.f);
            for (int e = 0; e < 4; ++e)
              if (i0 + e < len) {
                (&pv.x)[e] = a.p_in[i0 + e];
                (&ev.x)[e] = a.ea_in[i0 + e];
                (&sv.x)[e] = a.es_in[i0 + e];
              }
          }
          float* pp = &pv.x;
          float* ep = &ev.x;
          float* sp = &sv.x;
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int j = 4 * q + e;
            // g' = g - local_q + Q (optim.cpp:65); full band: local_q == g exactly
            const float gp = full_band ? d[j] : x[j] + d[j];
            const float ea = A.beta1 * ep[e] + A.one_minus_beta1 * gp;
            const float es = A.beta2 * sp[e] + A.one_minus_beta2 * gp * gp;
            float pnew = pp[e] - A.lr * adam_ratio(ea, es, A);
            if (A.lr_wd != 0.0f) pnew -= A.lr_wd * pnew;
            ep[e] = ea;
            sp[e] = es;
            pp[e] = pnew;
          }
          if (whole_out) {
            *reinterpret_cast<float4*>(a.p_out + i0) = pv;
            *reinterpret_cast<float4*>(a.ea_out + i0) = ev;
            *reinterpret_cast<float4*>(a.es_out + i0) = sv;
          } else {
            for (int e = 0; e < 4; ++e)
              if (i0 + e < len) {
                a.p_out[i0 + e] = pp[e];
                a.ea_out[i0 + e] = ep[e];
                a.es_out[i0 + e] = sp[e];
              }
          }
        }
      }
    } else {
      const bool exact_q = need_signs || dtype == DMB_FP16;
      if (MODE == ChunkMode::StepSgd) {
        // second inverse, Q = IDCT(wire values / 1): the A buffers are free once D2 is done
        named_sync(1 + grp, 128);
        store_row(a_hi, a_lo, t, exact_q, wire);
        fence_proxy_async_smem();
        named_sync(1 + grp, 128);
        if (t == 0) {
          tc_fence_after();
          issue_3x(tm + 128, ahi, alo, bthi, btlo, !exact_q);
          mma_commit(bar);
        }
      }
      // local_q (SGD / requested): full band -> exactly x
      float lq[64];
      if (need_lq) {
        load_tmem_row(tm_row + 64, lq);
      } else {
#pragma unroll
        for (int j = 0; j < 64; ++j) lq[j] = 0.0f;
      }
      if (full_band) {
#pragma unroll
        for (int j = 0; j < 64; ++j) lq[j] = x[j];
      }
      if (!skip) {
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          const uint64_t i0 = base + 4 * q;
          float4 mo = make_float4(x[4 * q] - lq[4 * q], x[4 * q + 1] - lq[4 * q + 1], x[4 * q + 2] - lq[4 * q + 2],
                                  x[4 * q + 3] - lq[4 * q + 3]);
          float4 lo4 = make_float4(lq[4 * q], lq[4 * q + 1], lq[4 * q + 2], lq[4 * q + 3]);
          float4 ma4 = make_float4(x[4 * q], x[4 * q + 1], x[4 * q + 2], x[4 * q + 3]);
          if (whole) {
            if (kSgd) *reinterpret_cast<float4*>(a.m_out + i0) = mo;
            if (a.local_q) *reinterpret_cast<float4*>(a.local_q + i0) = lo4;
            if (kSgd && a.m_accum) *reinterpret_cast<float4*>(a.m_accum + i0) = ma4;
          } else {
            for (int e = 0; e < 4; ++e)
              if (i0 + e < len) {
                if (kSgd) a.m_out[i0 + e] = (&mo.x)[e];
                if (a.local_q) a.local_q[i0 + e] = (&lo4.x)[e];
                if (kSgd && a.m_accum) a.m_accum[i0 + e] = (&ma4.x)[e];
              }
          }
        }
      }
      if (MODE == ChunkMode::StepSgd) {
        mbar_wait(bar, phase);
        phase ^= 1;
        tc_fence_after();
        float Q[64];
        load_tmem_row(tm_row + 128, Q);
        if (!skip) {
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            const uint64_t i0 = base + 4 * q;
            if (whole) {
              float4 pv = *reinterpret_cast<const float4*>(a.p_in + i0);
              pv.x -= a.sgd.lr * Q[4 * q];
              pv.y -= a.sgd.lr * Q[4 * q + 1];
              pv.z -= a.sgd.lr * Q[4 * q + 2];
              pv.w -= a.sgd.lr * Q[4 * q + 3];
              *reinterpret_cast<float4*>(a.p_out + i0) = pv;
            } else {
              for (int e = 0; e < 4; ++e)
                if (i0 + e < len) a.p_out[i0 + e] = a.p_in[i0 + e] - a.sgd.lr * Q[4 * q + e];
            }
          }
        }
      }
    }
    tc_fence_before();
    named_sync(1 + grp, 128);
  }

  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc(tmem_base, TMEM_COLS);
}

template <ChunkMode MODE>
void launch_mode(const ChunkArgs& a, cudaStream_t stream) {
  auto kern = demo_tc_kernel<MODE>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM_BYTES);
    attr = true;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const uint64_t ntiles = (a.geo.nchunks + TM - 1) / TM;
  const uint64_t ctas_needed = (ntiles + GROUPS - 1) / GROUPS;
  const unsigned grid = (unsigned)(ctas_needed < (uint64_t)sms ? (ctas_needed ? ctas_needed : 1) : sms);
  kern<<<grid, THREADS, SMEM_BYTES, stream>>>(a);
}

}  // namespace

bool tc_supported(ChunkMode mode, const ChunkArgs& a) {
  if (a.geo.s != S) return false;
  if (!(mode == ChunkMode::StepAdam || mode == ChunkMode::StepSgd || mode == ChunkMode::EncodeAdam ||
        mode == ChunkMode::EncodeSgd))
    return false;
  auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; };
  return al(a.g) && al(a.m_in) && al(a.m_out) && al(a.p_in) && al(a.p_out) && al(a.ea_in) && al(a.ea_out) &&
         al(a.es_in) && al(a.es_out) && al(a.local_q) && al(a.m_accum) && a.basis.Bhi != nullptr;
}

void launch_tc_kernel(ChunkMode mode, const ChunkArgs& a, cudaStream_t stream) {
  count_launches(1);
  switch (mode) {
    case ChunkMode::StepAdam: launch_mode<ChunkMode::StepAdam>(a, stream); break;
    case ChunkMode::StepSgd: launch_mode<ChunkMode::StepSgd>(a, stream); break;
    case ChunkMode::EncodeAdam: launch_mode<ChunkMode::EncodeAdam>(a, stream); break;
    case ChunkMode::EncodeSgd: launch_mode<ChunkMode::EncodeSgd>(a, stream); break;
    default: break;
  }
}

}  // namespace dmb
