// demo_chunk.cuh -- DeMo (DCT-TopK) prepare / merge / apply, warp per chunk.
//
// Generic SIMT path for every chunk size the reference accepts (s <= 1024).  It
// restates, per chunk of the shard:
//   momentum accumulate           optim.cpp:25-28           (EncodeSgd / StepSgd)
//   DctPlan::forward              transform.cpp:56-63       (FP32 FMA, basis from host FP64)
//   TopK, ties -> lower index     transform.cpp:127-135     (warp radix select)
//   certification + FP64 re-derivation of uncertain chunks (bit-exact indices)
//   condition_values + packing    replicate.cpp:137-144, :316-356
//   sparse inverse -> local_q     transform.cpp:137-147
//   m <- m - local_q              optim.cpp:35-37
//   decode_and_merge (DeMo)       replicate.cpp:282-309     (rank-ordered grid, /R, IDCT)
//   demo_sgd_apply / adamw_apply  optim.cpp:45-49, :57-74
//
// Lane l of a warp owns chunk elements / frequencies j = l + 32 e (e < E).  CH
// chunks are processed together so every basis element read from shared memory
// feeds CH FMAs.
#pragma once
#include <cfloat>

#include "dmb_internal.cuh"

namespace dmb {
namespace chunk_impl {

constexpr int kWarps = 8;
constexpr int kThreads = kWarps * 32;

// ---- warp TopK by MSB radix select over |c| bit patterns -------------------
// Finds the k largest keys, ties toward the lower index j = lane + 32 e.
template <int E, typename K>
__device__ __forceinline__ void warp_topk(const K (&key)[E], const bool (&valid)[E], int k,
                                          bool (&sel)[E]) {
  constexpr int kBits = sizeof(K) * 8 - 1;  // sign bit of |c| is always clear
  K T = 0;
  bool exact = false;  // count(key >= T) == k exactly: {key >= T} is the answer
#pragma unroll 1
  for (int b = kBits - 1; b >= 0; --b) {
    const K cand = T | (K(1) << b);
    int cnt = 0;
#pragma unroll
    for (int e = 0; e < E; ++e) cnt += __popc(__ballot_sync(kFull, valid[e] && key[e] >= cand));
    if (cnt >= k) {
      T = cand;
      if (cnt == k) {
        exact = true;
        break;
      }
    }
  }
  if (exact) {
#pragma unroll
    for (int e = 0; e < E; ++e) sel[e] = valid[e] && key[e] >= T;
    return;
  }
  // T is the k-th largest key; take every key > T and the lowest-index ties.
  int gt = 0;
#pragma unroll
  for (int e = 0; e < E; ++e) gt += __popc(__ballot_sync(kFull, valid[e] && key[e] > T));
  const int need = k - gt;
  int taken = 0;
  const unsigned lt = lanemask_lt();
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const unsigned eq = __ballot_sync(kFull, valid[e] && key[e] == T);
    const int rank = taken + __popc(eq & lt);
    sel[e] = valid[e] && (key[e] > T || (key[e] == T && rank < need));
    taken += __popc(eq);
  }
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(kFull, v, o));
  return v;
}
__device__ __forceinline__ float warp_min(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fminf(v, __shfl_xor_sync(kFull, v, o));
  return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

// Inverse over a sparse coefficient set held in registers: out[e] (i = l+32e)
// += sum over selected j ascending of coef_j * B[j][i] (transform.cpp:65-73 order).
template <int E>
__device__ __forceinline__ void sparse_inverse(const float (&coef)[E], const bool (&nz)[E],
                                               const float* B, int s, float (&out)[E]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int e = 0; e < E; ++e) out[e] = 0.0f;
#pragma unroll
  for (int eq = 0; eq < E; ++eq) {
    unsigned m = __ballot_sync(kFull, nz[eq]);
    while (m) {
      const int l = __ffs(m) - 1;
      m &= m - 1;
      const int j = l + 32 * eq;
      const float cj = __shfl_sync(kFull, coef[eq], l);
      const float* row = B + (size_t)j * s;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int i = lane + 32 * e;
        if (i < s) out[e] = fmaf(cj, row[i], out[e]);
      }
    }
  }
}

// FP64 re-derivation of one chunk with the oracle's exact operation order:
// acc = 0.0; for i ascending: acc = acc + B[j][i] * x_i (mul then add, no FMA),
// transform.cpp:56-63.  x is FP32 widened (the value the oracle is fed).
template <int E>
__device__ __forceinline__ void forward_fp64(const float (&x)[E], const double* B64, int s,
                                             double (&cd)[E]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int e = 0; e < E; ++e) cd[e] = 0.0;
#pragma unroll
  for (int e2 = 0; e2 < E; ++e2) {
    for (int l = 0; l < 32; ++l) {
      const int i = l + 32 * e2;
      if (i >= s) break;  // warp-uniform
      const double xi = (double)__shfl_sync(kFull, x[e2], l);
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int j = lane + 32 * e;
        if (j < s) cd[e] = __dadd_rn(cd[e], __dmul_rn(B64[(size_t)j * s + i], xi));
      }
    }
  }
}

template <int E, int CH, ChunkMode MODE>
__global__ void __launch_bounds__(kThreads) demo_chunk_kernel(const ChunkArgs a) {
  constexpr bool kEncode = MODE == ChunkMode::EncodeSgd || MODE == ChunkMode::EncodeAdam ||
                           MODE == ChunkMode::StepSgd || MODE == ChunkMode::StepAdam;
  constexpr bool kSgdMomentum = MODE == ChunkMode::EncodeSgd || MODE == ChunkMode::StepSgd;
  constexpr bool kMerge = MODE == ChunkMode::MergeSgd || MODE == ChunkMode::MergeAdam;
  constexpr bool kStep = MODE == ChunkMode::StepSgd || MODE == ChunkMode::StepAdam;
  constexpr bool kAdamApply = MODE == ChunkMode::StepAdam || MODE == ChunkMode::MergeAdam;

  extern __shared__ __align__(16) float smem[];
  const int s = a.geo.s;
  const int k = a.geo.k;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const bool smem_basis = s <= 64;

  if (kMerge || kStep) {
    if (step_failed(a.status)) return;  // state untouched after a TrainingError
  }
  if (a.list && *a.list_count == 0) return;  // nothing left uncertified

  float* sB = smem;
  float* sBT = smem + (smem_basis ? s * s : 0);
  float* grid_all = smem + (smem_basis ? 2 * s * s : 0);  // per warp: CH * 32E floats
  unsigned* flags_all = reinterpret_cast<unsigned*>(grid_all + kWarps * CH * 32 * E);
  if (smem_basis) {
    for (int t = threadIdx.x; t < s * s; t += blockDim.x) {
      sB[t] = a.basis.B[t];
      sBT[t] = a.basis.BT[t];
    }
    __syncthreads();
  }
  const float* B = smem_basis ? sB : a.basis.B;
  const float* BT = smem_basis ? sBT : a.basis.BT;
  float* grid = grid_all + warp * CH * 32 * E;
  unsigned* flags = flags_all + warp * CH * E;

  const uint64_t len = a.geo.len;
  const uint64_t nchunks = a.geo.nchunks;
  const uint64_t nvals = nchunks * (uint64_t)k;  // DeMo: C*k indices then C*k values
  const int dtype = a.geo.dtype;
  const bool sign_mode = a.geo.sign_mode;
  // certification bound: |c~_j - c_j| <= (s+3) u sqrt(2/s) ||x||_1  (u = 2^-24), see DESIGN.md
  const float eps_scale = (float)((s + 3) * 5.9604644775390625e-08 * sqrt(2.0 / s) * 1.01);

  const uint64_t warps_total = (uint64_t)gridDim.x * kWarps;
  const bool list_mode = a.list != nullptr;
  const uint64_t n_units = list_mode ? (uint64_t)*a.list_count : nchunks - a.first_chunk;
  for (uint64_t u0 = ((uint64_t)blockIdx.x * kWarps + warp) * CH; u0 < n_units; u0 += warps_total * CH) {
    const uint64_t c0 = list_mode ? (uint64_t)a.list[u0] : a.first_chunk + u0;  // list mode: CH == 1
    float x[CH][E];    // encode: v (m_acc or g); merge-adam: g
    float gv[CH][E];   // raw gradient (adam paths)
    float Q[CH][E];    // merged update
    float lq[CH][E];   // local_q
    bool in[CH][E];    // element exists (inside the shard)

    // ---- 1. inputs (coalesced: lanes walk consecutive elements of a chunk) ----
#pragma unroll
    for (int ch = 0; ch < CH; ++ch) {
      const uint64_t c = c0 + ch;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int i = lane + 32 * e;
        const uint64_t gi = c * (uint64_t)s + i;
        in[ch][e] = c < nchunks && i < s && gi < len;
        float g = 0.0f, m = 0.0f;
        if (in[ch][e]) {
          if (kEncode || MODE == ChunkMode::MergeAdam) g = a.g[gi];
          if (kSgdMomentum) m = a.m_in[gi];
        }
        if (kEncode && in[ch][e] && !isfinite(g)) latch_bad(a.status, gi);
        gv[ch][e] = g;
        // m = beta * m + g (optim.cpp:27): multiply, then add, no contraction
        x[ch][e] = kSgdMomentum ? __fadd_rn(__fmul_rn(a.sgd.beta, m), g) : g;
        if (kEncode && a.m_accum && in[ch][e]) a.m_accum[gi] = x[ch][e];
      }
    }

    // ---- 2. forward DCT for every chunk of the batch (FP32, basis in smem) ----
    float cf[CH][E];
    if (kEncode || MODE == ChunkMode::MergeAdam) {
#pragma unroll
      for (int ch = 0; ch < CH; ++ch)
#pragma unroll
        for (int e = 0; e < E; ++e) cf[ch][e] = 0.0f;
#pragma unroll
      for (int e2 = 0; e2 < E; ++e2) {
#pragma unroll 4
        for (int l = 0; l < 32; ++l) {
          const int i = l + 32 * e2;
          if (i >= s) break;  // warp-uniform
          float bt[E];
#pragma unroll
          for (int e = 0; e < E; ++e) {
            const int j = lane + 32 * e;
            bt[e] = j < s ? BT[(size_t)i * s + j] : 0.0f;
          }
#pragma unroll
          for (int ch = 0; ch < CH; ++ch) {
            const float xi = __shfl_sync(kFull, x[ch][e2], l);
#pragma unroll
            for (int e = 0; e < E; ++e) cf[ch][e] = fmaf(bt[e], xi, cf[ch][e]);
          }
        }
      }
    }

    // ---- 3. per chunk: selection, payload, local_q, merge, apply ----
#pragma unroll
    for (int ch = 0; ch < CH; ++ch) {
      const uint64_t c = c0 + ch;
      if (c >= nchunks) break;  // warp-uniform
      bool valid[E], sel[E];
#pragma unroll
      for (int e = 0; e < E; ++e) valid[e] = lane + 32 * e < s;
      float csel[E];  // coefficient carried by each selected frequency (FP32)

      if (kEncode) {
        if (k == s) {
#pragma unroll
          for (int e = 0; e < E; ++e) sel[e] = valid[e];
        } else {
          uint32_t key[E];
#pragma unroll
          for (int e = 0; e < E; ++e) key[e] = __float_as_uint(fabsf(cf[ch][e]));
          warp_topk<E, uint32_t>(key, valid, k, sel);
        }
        // certification: the selection (and, with signs on the wire, each sign) of
        // the FP32 coefficients provably equals the FP64 oracle's.
        float l1 = 0.0f;
#pragma unroll
        for (int e = 0; e < E; ++e) l1 += fabsf(x[ch][e]);
        l1 = warp_sum(l1);
        const float eps = eps_scale * l1;
        float kth = FLT_MAX, nxt = 0.0f;
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const float m = fabsf(cf[ch][e]);
          if (sel[e]) kth = fminf(kth, m);
          else if (valid[e]) nxt = fmaxf(nxt, m);
        }
        kth = warp_min(kth);
        nxt = warp_max(nxt);
        const bool need_signs = sign_mode || dtype == DMB_TERNARY;
        bool uncertain = k < s ? !(kth - nxt > 2.0f * eps) : (need_signs && !(kth > eps));
        if (isnan(l1)) uncertain = false;  // non-finite input: the step fails anyway
        if (a.force_fp64) uncertain = true;
        double cd[E];
        const bool fp64 = uncertain;
        if (fp64) {
          if (lane == 0) atomicAdd(&a.status->fallback_chunks, 1ull);
          forward_fp64<E>(x[ch], a.basis.B64, s, cd);
          if (k < s) {
            unsigned long long key[E];
#pragma unroll
            for (int e = 0; e < E; ++e)
              key[e] = (unsigned long long)__double_as_longlong(fabs(cd[e]));
            warp_topk<E, unsigned long long>(key, valid, k, sel);
          }
        }
        float wv[E];  // conditioned wire value of each selected frequency
#pragma unroll
        for (int e = 0; e < E; ++e) {
          csel[e] = fp64 ? (float)cd[e] : cf[ch][e];
          wv[e] = sel[e] ? (fp64 ? condition_f64(cd[e], dtype, sign_mode)
                                 : condition_f32(cf[ch][e], dtype, sign_mode))
                         : 0.0f;
        }

        // payload: ascending j within the chunk (transform.cpp:134)
        if (a.body) {
          uint32_t* idx_out = reinterpret_cast<uint32_t*>(a.body);
          uint8_t* val_out = a.body + nvals * 4;
          int before = 0;
          const unsigned lt = lanemask_lt();
#pragma unroll
          for (int e = 0; e < E; ++e) {
            const unsigned m = __ballot_sync(kFull, sel[e]);
            if (sel[e]) {
              const uint64_t t = c * (uint64_t)k + before + __popc(m & lt);
              idx_out[t] = (uint32_t)(lane + 32 * e);
              store_wire_value(val_out, t, wv[e], dtype);
            }
            before += __popc(m);
          }
        }

        // one-rank AdamW step without a local_q output: g' = g - local_q + Q needs only
        // IDCT(wire - coef) over the selection, one sparse inverse instead of two
        const bool fused_w = MODE == ChunkMode::StepAdam && !a.local_q && k < s;
        // local_q (unsigned coefficients, SPEC: sign never touches local state)
        if (fused_w) {
          float wd[E];
#pragma unroll
          for (int e = 0; e < E; ++e) wd[e] = sel[e] ? wv[e] - csel[e] : 0.0f;
          sparse_inverse<E>(wd, sel, B, s, Q[ch]);
#pragma unroll
          for (int e = 0; e < E; ++e) lq[ch][e] = 0.0f;
        } else if (k == s) {
#pragma unroll
          for (int e = 0; e < E; ++e) lq[ch][e] = x[ch][e];  // exact copy, transform.cpp:119-125
        } else {
          sparse_inverse<E>(csel, sel, B, s, lq[ch]);
        }

        if (kSgdMomentum) {
#pragma unroll
          for (int e = 0; e < E; ++e) {
            const uint64_t gi = c * (uint64_t)s + lane + 32 * e;
            if (in[ch][e]) a.m_out[gi] = x[ch][e] - lq[ch][e];
          }
        }
        if (a.local_q) {
#pragma unroll
          for (int e = 0; e < E; ++e) {
            const uint64_t gi = c * (uint64_t)s + lane + 32 * e;
            if (in[ch][e]) a.local_q[gi] = lq[ch][e];
          }
        }
        if (kStep && !fused_w) {
          // merge of a one-member group: grid = conditioned values / 1, then IDCT
          bool nz[E];
#pragma unroll
          for (int e = 0; e < E; ++e) nz[e] = wv[e] != 0.0f;
          sparse_inverse<E>(wv, nz, B, s, Q[ch]);
        }
      }

      if (kMerge) {
        // decode_and_merge, DeMo branch (replicate.cpp:282-309): rank-ordered grid
        float* gch = grid + ch * 32 * E;
#pragma unroll
        for (int e = 0; e < E; ++e) gch[lane + 32 * e] = 0.0f;
        __syncwarp();
        for (int r = 0; r < a.in.R; ++r) {
          const uint32_t* idx_r = reinterpret_cast<const uint32_t*>(a.in.body[r]);
          const uint8_t* val_r = a.in.body[r] + nvals * 4;
          for (int t = lane; t < k; t += 32) {
            const uint64_t tt = c * (uint64_t)k + t;
            const uint32_t j = idx_r[tt];
            if (j >= (uint32_t)s) {
              atomicExch(&a.status->protocol_error, 1u);
              continue;
            }
            gch[j] += load_wire_value(val_r, tt, dtype);
          }
          __syncwarp();
        }
        float gval[E];
        bool nz[E];
        const float R = (float)a.in.R;
#pragma unroll
        for (int e = 0; e < E; ++e) {
          gval[e] = valid[e] ? gch[lane + 32 * e] / R : 0.0f;
          nz[e] = gval[e] != 0.0f;  // DctPlan::inverse skips zero coefficients
        }
        __syncwarp();
        sparse_inverse<E>(gval, nz, B, s, Q[ch]);

        if (MODE == ChunkMode::MergeAdam) {
          // local_q re-derived from g and this rank's own indices (no stored copy)
          if (k == s) {
#pragma unroll
            for (int e = 0; e < E; ++e) lq[ch][e] = x[ch][e];
          } else {
            unsigned* f = flags + ch * E;
#pragma unroll
            for (int e = 0; e < E; ++e)
              if (lane == 0) f[e] = 0u;
            __syncwarp();
            const uint32_t* idx_o = reinterpret_cast<const uint32_t*>(a.in.body[a.own_rank]);
            for (int t = lane; t < k; t += 32) {
              const uint32_t j = idx_o[c * (uint64_t)k + t];
              if (j < (uint32_t)s) atomicOr(&f[j >> 5], 1u << (j & 31));
            }
            __syncwarp();
            bool own[E];
#pragma unroll
            for (int e = 0; e < E; ++e) own[e] = (f[e] >> lane) & 1u;
            __syncwarp();
            sparse_inverse<E>(cf[ch], own, B, s, lq[ch]);
          }
        }
      }

      // ---- apply ----
      if (MODE == ChunkMode::StepSgd || MODE == ChunkMode::MergeSgd) {
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const uint64_t gi = c * (uint64_t)s + lane + 32 * e;
          if (!in[ch][e]) continue;
          if (a.q_out) a.q_out[gi] = Q[ch][e];
          if (a.p_out) a.p_out[gi] = a.p_in[gi] - a.sgd.lr * Q[ch][e];
        }
      }
      if (kAdamApply) {
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const uint64_t gi = c * (uint64_t)s + lane + 32 * e;
          if (!in[ch][e]) continue;
          if (a.q_out) a.q_out[gi] = Q[ch][e];
          const AdamScalars& A = a.adam;
          const float gp = (gv[ch][e] - lq[ch][e]) + Q[ch][e];  // optim.cpp:65
          const float ea = A.beta1 * a.ea_in[gi] + A.one_minus_beta1 * gp;
          const float es = A.beta2 * a.es_in[gi] + A.one_minus_beta2 * gp * gp;
          float p = a.p_in[gi] - A.lr * adam_ratio(ea, es, A);
          if (A.lr_wd != 0.0f) p -= A.lr_wd * p;
          a.ea_out[gi] = ea;
          a.es_out[gi] = es;
          a.p_out[gi] = p;
        }
      }
    }
  }
}

template <int E, int CH, ChunkMode MODE>
void launch_t(const ChunkArgs& a, cudaStream_t stream) {
  count_launches(1);
  const int s = a.geo.s;
  const size_t basis = s <= 64 ? 2u * s * s * sizeof(float) : 0;
  const size_t smem = basis + (size_t)kWarps * CH * 32 * E * sizeof(float) +
                      (size_t)kWarps * CH * E * sizeof(unsigned);
  auto kern = demo_chunk_kernel<E, CH, MODE>;
  if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const uint64_t units = (a.geo.nchunks - a.first_chunk + (uint64_t)kWarps * CH - 1) / ((uint64_t)kWarps * CH);
  uint64_t grid = (uint64_t)sms * 4;
  if (units < grid) grid = units ? units : 1;
  if (a.list) {  // list length lives on the device: fill every SM to its occupancy limit
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, smem);
    grid = (uint64_t)sms * (uint64_t)(per_sm > 0 ? per_sm : 1);
  }
  kern<<<(unsigned)grid, kThreads, smem, stream>>>(a);
}

}  // namespace chunk_impl
}  // namespace dmb
