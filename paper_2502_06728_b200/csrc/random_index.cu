// random_index.cu -- the Random scheme's index set on the device, bit-exact with
// selected_indices (replicate.cpp:160-172):
//
//   all = iota(L); Rng rng(mix_seed(seed, step, shard));   // engine = mt19937_64(mix64(.))
//   for i = L .. 2: j = rng.below(i); swap(all[i-1], all[j])  // rng.hpp:40-45, rng.cpp:27-37
//   idx = sort(all[0 .. count))
//
// Only the iterations i = L .. count+1 decide WHICH values end in positions
// [0, count); the later ones permute that prefix among itself and the result is
// sorted anyway.  So (1) one CTA draws j_i for those L - count iterations from the
// MT19937-64 stream (block-parallel twist, Lemire debias with an exact sequential
// fix-up when a rejection occurs); (2) for every position t, first[t]/second[t]
// hold the two smallest iterations that targeted it (atomicMin passes); (3) the
// value that ends in position x < count is resolved by following
//   D(i) = value at position i-1 just before iteration i
//        = D(min{i' > i : j_i' = i-1})  or  i-1 if there is none
// from i* = first[x]; (4) selected values are marked in a bitmap and compacted in
// ascending order (no sort).  Nothing here runs on the host.
#include "dmb_internal.cuh"

namespace dmb {
namespace {

constexpr uint32_t kNone = 0xffffffffu;
constexpr int kMtN = 312;
constexpr int kMtThreads = 320;

__device__ __forceinline__ uint64_t temper(uint64_t y) {
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

__device__ __forceinline__ uint64_t twist_word(uint64_t cur, uint64_t next, uint64_t far) {
  const uint64_t y = (cur & 0xFFFFFFFF80000000ULL) | (next & 0x7FFFFFFFULL);
  return far ^ (y >> 1) ^ ((y & 1ULL) ? 0xB5026F5AA96619E9ULL : 0ULL);
}

// draws[d] = below(len - d) for d in [0, ndraws), consuming the engine in order.
__global__ void __launch_bounds__(kMtThreads) mt_draws_kernel(uint64_t engine_seed, uint64_t len,
                                                              uint64_t ndraws,
                                                              uint32_t* __restrict__ draws) {
  __shared__ uint64_t mt[kMtN];
  __shared__ int any_reject;
  __shared__ uint64_t d_shared;
  const int t = threadIdx.x;
  if (t == 0) {
    // std::mt19937_64 seeding (f = 6364136223846793005)
    uint64_t v = engine_seed;
    mt[0] = v;
    for (int i = 1; i < kMtN; ++i) {
      v = 6364136223846793005ULL * (v ^ (v >> 62)) + (uint64_t)i;
      mt[i] = v;
    }
    d_shared = 0;
  }
  __syncthreads();
  uint64_t d0 = 0;
  while (d0 < ndraws) {
    // ---- twist: k < 156 from old words, 156 <= k < 311 from new, then k = 311 ----
    uint64_t nv = 0;
    if (t < 156) nv = twist_word(mt[t], mt[t + 1], mt[t + 156]);
    __syncthreads();
    if (t < 156) mt[t] = nv;
    __syncthreads();
    if (t >= 156 && t < 311) nv = twist_word(mt[t], mt[t + 1], mt[t - 156]);
    __syncthreads();
    if (t >= 156 && t < 311) mt[t] = nv;
    __syncthreads();
    if (t == 0) {
      mt[311] = twist_word(mt[311], mt[0], mt[155]);
      any_reject = 0;
    }
    __syncthreads();
    // ---- Lemire below(n), n = len - d: accept unless low64(x*n) < (2^64 - n) % n ----
    uint64_t x = 0;
    uint32_t hi = 0;
    bool mine = false;
    if (t < kMtN) {
      x = temper(mt[t]);
      const uint64_t d = d0 + t;
      if (d < ndraws) {
        mine = true;
        const uint64_t n = len - d;
        const uint64_t lo = x * n;
        hi = (uint32_t)__umul64hi(x, n);
        if (lo < n) {  // the threshold is < n: only then can it reject
          const uint64_t threshold = (0ULL - n) % n;
          if (lo < threshold) any_reject = 1;
        }
      }
    }
    __syncthreads();
    if (!any_reject) {
      if (mine) draws[d0 + t] = hi;
      d0 += kMtN;
    } else {
      // exact sequential replay of this batch: a rejection consumes an output
      // without producing a draw, shifting every later draw by one
      if (t == 0) {
        uint64_t d = d0;
        for (int q = 0; q < kMtN && d < ndraws; ++q) {
          const uint64_t xx = temper(mt[q]);
          const uint64_t n = len - d;
          const uint64_t lo = xx * n;
          if (lo < n && lo < (0ULL - n) % n) continue;
          draws[d] = (uint32_t)__umul64hi(xx, n);
          ++d;
        }
        d_shared = d;
      }
      __syncthreads();
      d0 = d_shared;
    }
    __syncthreads();
  }
}

__global__ void first_pass(const uint32_t* __restrict__ draws, uint64_t len, uint64_t ndraws,
                           uint32_t* __restrict__ first) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t d = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; d < ndraws; d += stride)
    atomicMin(&first[draws[d]], (uint32_t)(len - d));
}

__global__ void second_pass(const uint32_t* __restrict__ draws, uint64_t len, uint64_t ndraws,
                            const uint32_t* __restrict__ first, uint32_t* __restrict__ second) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t d = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; d < ndraws; d += stride) {
    const uint32_t tgt = draws[d];
    const uint32_t it = (uint32_t)(len - d);
    if (first[tgt] != it) atomicMin(&second[tgt], it);
  }
}

__global__ void resolve_kernel(uint64_t count, const uint32_t* __restrict__ first,
                               const uint32_t* __restrict__ second, uint32_t* __restrict__ bitmap) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t x = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; x < count; x += stride) {
    uint32_t v = (uint32_t)x;
    uint32_t i = first[x];
    while (i != kNone) {  // follow D(i)
      const uint32_t pos = i - 1;
      const uint32_t f = first[pos];
      const uint32_t nxt = f == i ? second[pos] : f;
      v = pos;
      i = nxt;
    }
    atomicOr(&bitmap[v >> 5], 1u << (v & 31));
  }
}

// exclusive popcount prefix over bitmap words: per-block partials, then a single
// block scans the partials, then per-word ranks
constexpr int kScanBlock = 1024;

__global__ void __launch_bounds__(kScanBlock) block_popc(const uint32_t* __restrict__ bitmap,
                                                         uint64_t words, uint32_t* __restrict__ partial) {
  __shared__ uint32_t warp_sums[32];
  const uint64_t w = (uint64_t)blockIdx.x * kScanBlock + threadIdx.x;
  uint32_t v = w < words ? __popc(bitmap[w]) : 0;
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  if ((threadIdx.x & 31) == 0) warp_sums[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    uint32_t s = warp_sums[threadIdx.x];
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
    if (threadIdx.x == 0) partial[blockIdx.x] = s;
  }
}

__global__ void __launch_bounds__(kScanBlock) scan_partials(uint32_t* __restrict__ partial, uint64_t n) {
  // single block, sequential over tiles of 1024: exclusive scan in place
  __shared__ uint32_t buf[kScanBlock];
  __shared__ uint32_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (uint64_t base = 0; base < n; base += kScanBlock) {
    const uint64_t i = base + threadIdx.x;
    const uint32_t v = i < n ? partial[i] : 0;
    buf[threadIdx.x] = v;
    __syncthreads();
    for (int o = 1; o < kScanBlock; o <<= 1) {
      const uint32_t add = threadIdx.x >= (unsigned)o ? buf[threadIdx.x - o] : 0;
      __syncthreads();
      buf[threadIdx.x] += add;
      __syncthreads();
    }
    if (i < n) partial[i] = carry + buf[threadIdx.x] - v;
    __syncthreads();
    if (threadIdx.x == kScanBlock - 1) carry += buf[kScanBlock - 1];
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kScanBlock) word_ranks(const uint32_t* __restrict__ bitmap, uint64_t words,
                                                         const uint32_t* __restrict__ partial,
                                                         uint32_t* __restrict__ rank,
                                                         uint32_t* __restrict__ idx) {
  __shared__ uint32_t warp_sums[32];
  const uint64_t w = (uint64_t)blockIdx.x * kScanBlock + threadIdx.x;
  const uint32_t bits = w < words ? bitmap[w] : 0;
  const uint32_t v = __popc(bits);
  // block exclusive scan
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t inc = v;
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t n = __shfl_up_sync(kFull, inc, o);
    if (lane >= o) inc += n;
  }
  if (lane == 31) warp_sums[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    uint32_t s = warp_sums[lane];
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t n = __shfl_up_sync(kFull, s, o);
      if (lane >= o) s += n;
    }
    warp_sums[lane] = s;
  }
  __syncthreads();
  const uint32_t excl = partial[blockIdx.x] + (warp ? warp_sums[warp - 1] : 0) + inc - v;
  if (w < words) {
    rank[w] = excl;
    uint32_t b = bits, r = excl;
    while (b) {
      const int pos = __ffs(b) - 1;
      b &= b - 1;
      idx[r++] = (uint32_t)(w * 32 + pos);
    }
  }
}

__global__ void fill_prefix(uint32_t* __restrict__ bitmap, uint64_t len) {
  // count == len: every element is selected
  const uint64_t words = (len + 31) / 32;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; w < words; w += stride) {
    const uint64_t lo = w * 32;
    const uint64_t n = len - lo < 32 ? len - lo : 32;
    bitmap[w] = n == 32 ? 0xffffffffu : ((1u << n) - 1u);
  }
}

unsigned sm_grid(uint64_t n, int block) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const uint64_t want = (n + block - 1) / block;
  const uint64_t cap = (uint64_t)sms * 8;
  return (unsigned)(want < cap ? (want ? want : 1) : cap);
}

}  // namespace

void launch_random_indices(uint64_t engine_seed, uint64_t len, uint64_t count,
                           const RandomScratch& s, cudaStream_t stream) {
  count_launches(len > count ? 7 : 4);
  const uint64_t words = (len + 31) / 32;
  cudaMemsetAsync(s.bitmap, 0, words * sizeof(uint32_t), stream);
  if (count >= len) {
    fill_prefix<<<sm_grid(words, 256), 256, 0, stream>>>(s.bitmap, len);
  } else {
    const uint64_t ndraws = len - count;
    mt_draws_kernel<<<1, kMtThreads, 0, stream>>>(engine_seed, len, ndraws, s.draws);
    cudaMemsetAsync(s.first, 0xff, len * sizeof(uint32_t), stream);
    cudaMemsetAsync(s.second, 0xff, len * sizeof(uint32_t), stream);
    first_pass<<<sm_grid(ndraws, 256), 256, 0, stream>>>(s.draws, len, ndraws, s.first);
    second_pass<<<sm_grid(ndraws, 256), 256, 0, stream>>>(s.draws, len, ndraws, s.first, s.second);
    resolve_kernel<<<sm_grid(count, 256), 256, 0, stream>>>(count, s.first, s.second, s.bitmap);
  }
  const uint64_t blocks = (words + kScanBlock - 1) / kScanBlock;
  uint32_t* partial = s.rank + words + 1;  // scratch tail of the rank array
  block_popc<<<(unsigned)blocks, kScanBlock, 0, stream>>>(s.bitmap, words, partial);
  scan_partials<<<1, kScanBlock, 0, stream>>>(partial, blocks);
  word_ranks<<<(unsigned)blocks, kScanBlock, 0, stream>>>(s.bitmap, words, partial, s.rank, s.idx);
}

}  // namespace dmb
