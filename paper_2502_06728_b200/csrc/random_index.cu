// random_index.cu -- the Random scheme's index set on the device, bit-exact with
// selected_indices (replicate.cpp:160-172):
//
//   all = iota(L); Rng rng(mix_seed(seed, step, shard));   // engine = mt19937_64(mix64(.))
//   for i = L .. 2: j = rng.below(i); swap(all[i-1], all[j])  // rng.hpp:40-45, rng.cpp:27-37
//   idx = sort(all[0 .. count))
//
// Only the iterations i = L .. count+1 decide WHICH values end in positions
// [0, count); the later ones permute that prefix among itself and the result is
// sorted anyway.  So (1) the draws j_i of those L - count iterations come from the
// MT19937-64 stream split into one wave of substreams (two per CTA), every
// substream started by a GF(2) jump-ahead (below); Lemire's debias rejects an output with
// probability < 2^-32, and a rejection shifts every later draw by one output, so the CTAs
// assume none and report the first output that could be one -- an exact sequential
// replay from that substream fixes the rare case; (2) for every position t, first[t]/second[t]
// hold the two smallest iterations that targeted it (one atomicMin pass); (3) the
// value that ends in position x < count is resolved by following
//   D(i) = value at position i-1 just before iteration i
//        = D(min{i' > i : j_i' = i-1})  or  i-1 if there is none
// from i* = first[x]; (4) selected values are marked in a bitmap and compacted in
// ascending order (no sort).
//
// Jump-ahead.  One engine output advances the state window (x_i .. x_i+311) by one word:
// a linear map T over GF(2) whose characteristic polynomial phi (degree 19937) is found once
// per process by Berlekamp-Massey on the engine's own output bits.  With
// P_b(x) = x^(b W) mod phi (seed independent, computed once on the host and cached), the
// window at output b W is  P_b(T) s0 = XOR over the set coefficients i of P_b of the window
// (x_i .. x_i+311)  -- a correlation of P_b's bits with the first 20 k words of the seeded
// engine, which one CTA computes in shared memory.  It differs from T^(bW) s0 at most in
// the 31 low bits of the window's first word, which the twist never reads (only its upper
// 33 bits enter y), so every output of the substream is exact.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "dmb_internal.cuh"

namespace dmb {
namespace {

constexpr uint32_t kNone = 0xffffffffu;
constexpr int kMtN = 312;
constexpr int kMtThreads = 320;

__host__ __device__ __forceinline__ uint64_t temper(uint64_t y) {
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

__host__ __device__ __forceinline__ uint64_t twist_word(uint64_t cur, uint64_t next, uint64_t far) {
  const uint64_t y = (cur & 0xFFFFFFFF80000000ULL) | (next & 0x7FFFFFFFULL);
  return far ^ (y >> 1) ^ ((y & 1ULL) ? 0xB5026F5AA96619E9ULL : 0ULL);
}

// one in-place twist of the 312-word window by kMtThreads threads (two dependent halves)
__device__ __forceinline__ void twist_block(uint64_t* mt, int t) {
  uint64_t nv = 0;
  if (t < 156) nv = twist_word(mt[t], mt[t + 1], mt[t + 156]);
  __syncthreads();
  if (t < 156) mt[t] = nv;
  __syncthreads();
  if (t >= 156 && t < 311) nv = twist_word(mt[t], mt[t + 1], mt[t - 156]);
  __syncthreads();
  if (t >= 156 && t < 311) mt[t] = nv;
  __syncthreads();
  if (t == 0) mt[311] = twist_word(mt[311], mt[0], mt[155]);
  __syncthreads();
}

// std::mt19937_64 seeding (f = 6364136223846793005), then the first 64 twists: seq holds the
// words x_0 .. x_{kMtSeqWords-1} of the engine (the window at output i is seq[i .. i+311])
__global__ void __launch_bounds__(kMtThreads) mt_seq_kernel(uint64_t engine_seed, uint64_t* __restrict__ seq) {
  __shared__ uint64_t mt[kMtN];
  const int t = threadIdx.x;
  if (t == 0) {
    uint64_t v = engine_seed;
    mt[0] = v;
    for (int i = 1; i < kMtN; ++i) {
      v = 6364136223846793005ULL * (v ^ (v >> 62)) + (uint64_t)i;
      mt[i] = v;
    }
  }
  __syncthreads();
  if (t < kMtN) seq[t] = mt[t];
  for (uint64_t tw = 1; tw * kMtN < kMtSeqWords; ++tw) {
    twist_block(mt, t);
    if (t < kMtN) seq[tw * kMtN + t] = mt[t];
  }
}

// Lemire below(n) on output x: the draw, and whether the output could be rejected
__device__ __forceinline__ uint32_t lemire(uint64_t x, uint64_t n, bool& rejected) {
  const uint64_t lo = x * n;
  rejected = lo < n && lo < (0ULL - n) % n;  // the threshold (2^64 - n) mod n is < n
  return (uint32_t)__umul64hi(x, n);
}

// Substreams: W outputs each (a multiple of 312), kSubPerCta per CTA (their twists share the
// CTA's barriers).  Substream b: window P_b(T) s0 by correlation, then W / 312 twists on
// ping-pong windows (two barriers per twist); draw d = output o (no rejection before o
// assumed; the first output that could be one is reported in *reject)
constexpr int kSubPerCta = 1;
constexpr int kCorrGroups = 2;  // thread groups sharing one substream's correlation
constexpr int kBlockThreads = kCorrGroups * kMtThreads;
constexpr uint16_t kZeroPos = (uint16_t)kMtSeqWords;  // a term list's padding: words past the sequence, zero

__global__ void __launch_bounds__(kBlockThreads) mt_block_kernel(const uint64_t* __restrict__ seq,
                                                                 const uint16_t* __restrict__ pos,
                                                                 const uint32_t* __restrict__ pos_off, uint64_t W,
                                                                 uint64_t nsub, uint64_t len, uint64_t ndraws,
                                                                 uint32_t* __restrict__ draws,
                                                                 uint64_t* __restrict__ windows,
                                                                 unsigned long long* __restrict__ reject) {
  extern __shared__ uint64_t sm[];
  uint64_t* xs = sm;                               // the engine's first kMtSeqWords words, then kMtN zeros
  uint64_t* win = xs + kMtSeqWords + kMtN;         // [2][312]: ping-pong windows
  uint64_t* part = win + 2 * kMtN;                 // [312]: the second group's half of the correlation
  const int grp = threadIdx.x / kMtThreads, t = threadIdx.x % kMtThreads;
  const uint64_t b = blockIdx.x;
  const bool live = b < nsub && t < kMtN && grp == 0;
  for (uint64_t i = threadIdx.x; i < kMtSeqWords; i += kBlockThreads) xs[i] = seq[i];
  for (int i = threadIdx.x; i < kMtN; i += kBlockThreads) xs[kMtSeqWords + i] = 0ull;
  __syncthreads();
  uint64_t* w0 = win;
  uint64_t acc = 0;
  if (b < nsub && t < kMtN) {
    // the correlation: word t of the window = XOR over the exponents i of P_b's terms of the
    // engine word t + i.  The exponents come as a list (16 bits each, four per load; the last
    // group padded with kZeroPos, which reads zeros), four independent accumulators keep four
    // loads in flight, the two thread groups take alternate groups of four terms
    const uint64_t* pq = reinterpret_cast<const uint64_t*>(pos + pos_off[b]);
    const uint32_t nq = (pos_off[b + 1] - pos_off[b]) / 4;
    const uint64_t* xt = xs + t;
    uint64_t a0 = 0, a1 = 0, a2 = 0, a3 = 0;
    for (uint32_t q = grp; q < nq; q += kCorrGroups) {  // uniform within a group: broadcast loads
      const uint64_t w = __ldg(pq + q);
      a0 ^= xt[(uint32_t)(w & 0xffffu)];
      a1 ^= xt[(uint32_t)((w >> 16) & 0xffffu)];
      a2 ^= xt[(uint32_t)((w >> 32) & 0xffffu)];
      a3 ^= xt[(uint32_t)(w >> 48)];
    }
    acc = (a0 ^ a1) ^ (a2 ^ a3);
    if (grp) part[t] = acc;
  }
  __syncthreads();
  if (live) {
    const uint64_t win0 = acc ^ part[t];
    w0[t] = win0;
    windows[b * kMtN + t] = win0;
  }
  const uint64_t twists = W / kMtN;
  const uint64_t o0 = b * W;
  for (uint64_t tw = 0; tw < twists; ++tw) {
    const uint64_t* cur = w0 + (tw & 1) * kMtN;
    uint64_t* nxt = w0 + ((tw + 1) & 1) * kMtN;
    __syncthreads();  // cur complete (previous twist or the correlation)
    if (grp == 0 && t < 156) nxt[t] = twist_word(cur[t], cur[t + 1], cur[t + 156]);
    __syncthreads();
    if (grp == 0 && t >= 156 && t < 311) nxt[t] = twist_word(cur[t], cur[t + 1], nxt[t - 156]);
    if (grp == 0 && t == 311) nxt[311] = twist_word(cur[311], nxt[0], nxt[155]);
    __syncthreads();
    const uint64_t o = o0 + tw * kMtN + t;
    if (live && o < ndraws) {
      bool rej;
      draws[o] = lemire(temper(nxt[t]), len - o, rej);
      if (rej) atomicMin(reject, (unsigned long long)o);
    }
  }
}

// The rare case: an output from *reject on was rejected, so every later draw moves by one
// output.  Replay from the start of that substream, sequentially from the rejection on.
__global__ void __launch_bounds__(kMtThreads) mt_fixup_kernel(const uint64_t* __restrict__ windows, uint64_t W,
                                                              uint64_t len, uint64_t ndraws,
                                                              uint32_t* __restrict__ draws,
                                                              const unsigned long long* __restrict__ reject) {
  __shared__ uint64_t mt[kMtN];
  __shared__ uint64_t d_shared;
  const uint64_t ostar = *reject;
  if (ostar >= ndraws) return;
  const int t = threadIdx.x;
  const uint64_t b = ostar / W;
  if (t < kMtN) mt[t] = windows[b * kMtN + t];
  uint64_t o = b * W, d = o;  // no rejection before ostar: draw = output there
  if (t == 0) d_shared = d;
  __syncthreads();
  while (d < ndraws) {
    twist_block(mt, t);
    if (t == 0) {
      for (int q = 0; q < kMtN && d < ndraws; ++q, ++o) {
        if (o < ostar) {  // unaffected: already written by mt_block_kernel
          ++d;
          continue;
        }
        bool rej;
        const uint32_t v = lemire(temper(mt[q]), len - d, rej);
        if (rej) continue;  // consumed without a draw
        draws[d++] = v;
      }
      d_shared = d;
    }
    __syncthreads();
    d = d_shared;  // o advances in thread 0 only; the loop condition uses d
    __syncthreads();
  }
}

// ---- host: GF(2)[x] arithmetic for the jump polynomials ----
constexpr int kDeg = 19937;
constexpr int kPW = kMtN;  // words of a reduced polynomial (degree < 19937)

struct DevPositions {
  uint16_t* pos = nullptr;      // the exponents of every P_b's terms, groups of four (kZeroPos pad)
  uint32_t* off = nullptr;      // [b]: start of P_b's list in pos; [blocks]: the end
  uint64_t blocks = 0;
};
struct JumpSet {
  std::vector<std::vector<uint64_t>> polys;  // x^(b W) mod phi, b = 0, 1, ...
  std::map<int, DevPositions> dev;           // device copies (term lists)
};
struct JumpTable {
  std::mutex mu;
  bool ready = false;
  std::vector<uint64_t> phish;   // 64 x (kPW + 1) words: phi << s, s = 0..63
  std::map<uint64_t, JumpSet> sets;  // by substream length W
  std::string error;
};
JumpTable& jump_table() {
  static JumpTable t;
  return t;
}

inline int bit(const std::vector<uint64_t>& v, uint64_t i) { return (int)((v[i >> 6] >> (i & 63)) & 1u); }

// reduce a product (up to degree 2 * 19936) modulo phi in place; result in words [0, kPW)
void reduce(std::vector<uint64_t>& p, const std::vector<uint64_t>& phish) {
  for (int64_t k = (int64_t)p.size() * 64 - 1; k >= kDeg; --k) {
    if (!((p[k >> 6] >> (k & 63)) & 1u)) continue;
    const uint64_t sh = (uint64_t)(k - kDeg);
    const uint64_t w = sh >> 6, s = sh & 63;
    const uint64_t* ph = &phish[s * (kPW + 1)];
    for (int q = 0; q <= kPW && w + q < p.size(); ++q) p[w + q] ^= ph[q];
  }
  p.resize(kPW);
}

std::vector<uint64_t> mulmod(const std::vector<uint64_t>& a, const std::vector<uint64_t>& b,
                             const std::vector<uint64_t>& phish) {
  std::vector<uint64_t> bsh((size_t)64 * (kPW + 1));  // b << s
  for (int s = 0; s < 64; ++s)
    for (int q = 0; q <= kPW; ++q) {
      const uint64_t lo = q < kPW ? b[q] << s : 0;
      const uint64_t hi = (q > 0 && s) ? b[q - 1] >> (64 - s) : 0;
      bsh[(size_t)s * (kPW + 1) + q] = lo | hi;
    }
  std::vector<uint64_t> p(2 * kPW + 2, 0);
  for (int w = 0; w < kPW; ++w) {
    uint64_t bits = a[w];
    while (bits) {
      const int s = __builtin_ctzll(bits);
      bits &= bits - 1;
      const uint64_t* src = &bsh[(size_t)s * (kPW + 1)];
      for (int q = 0; q <= kPW; ++q) p[w + q] ^= src[q];
    }
  }
  reduce(p, phish);
  return p;
}

std::vector<uint64_t> sqrmod(const std::vector<uint64_t>& a, const std::vector<uint64_t>& phish) {
  auto spread = [](uint32_t x) {  // bit i -> bit 2i
    uint64_t v = x;
    v = (v | (v << 16)) & 0x0000FFFF0000FFFFull;
    v = (v | (v << 8)) & 0x00FF00FF00FF00FFull;
    v = (v | (v << 4)) & 0x0F0F0F0F0F0F0F0Full;
    v = (v | (v << 2)) & 0x3333333333333333ull;
    v = (v | (v << 1)) & 0x5555555555555555ull;
    return v;
  };
  std::vector<uint64_t> p(2 * kPW + 2, 0);
  for (int w = 0; w < kPW; ++w) {
    p[2 * w] = spread((uint32_t)a[w]);
    p[2 * w + 1] = spread((uint32_t)(a[w] >> 32));
  }
  reduce(p, phish);
  return p;
}

std::vector<uint64_t> powmod(std::vector<uint64_t> base, uint64_t e, const std::vector<uint64_t>& phish) {
  std::vector<uint64_t> r(kPW, 0);
  r[0] = 1;
  while (e) {
    if (e & 1) r = mulmod(r, base, phish);
    e >>= 1;
    if (e) base = sqrmod(base, phish);
  }
  return r;
}

// phi by Berlekamp-Massey on the most significant bit of the engine's words x_312, x_313, ...
bool build_phi(JumpTable& J) {
  const int N = 2 * kDeg + 64;
  std::vector<uint64_t> mt(kMtN);
  uint64_t v = 5489;
  mt[0] = v;
  for (int i = 1; i < kMtN; ++i) {
    v = 6364136223846793005ULL * (v ^ (v >> 62)) + (uint64_t)i;
    mt[i] = v;
  }
  std::vector<uint8_t> s(N);
  for (int n = 0, pos = kMtN; n < N; ++n, ++pos) {
    if (pos == kMtN) {
      for (int k = 0; k < kMtN; ++k) mt[k] = twist_word(mt[k], mt[(k + 1) % kMtN], mt[(k + 156) % kMtN]);
      pos = 0;
    }
    s[n] = (uint8_t)(mt[pos] >> 63);
  }
  const int W = N / 64 + 2;
  std::vector<uint64_t> R(W + 2, 0), Cp(W + 2, 0), Bp(W + 2, 0), T;
  for (int t = 0; t < N; ++t)  // R[t] = s[N - 1 - t]
    if (s[N - 1 - t]) R[t >> 6] |= 1ull << (t & 63);
  Cp[0] = Bp[0] = 1;
  int L = 0, m = 1;
  auto window = [&](uint64_t off) {  // 64 bits of R from bit off
    const uint64_t w = off >> 6, sh = off & 63;
    const uint64_t lo = w < R.size() ? R[w] : 0, hi = w + 1 < R.size() ? R[w + 1] : 0;
    return sh ? (lo >> sh) | (hi << (64 - sh)) : lo;
  };
  for (int n = 0; n < N; ++n) {
    const uint64_t off = (uint64_t)(N - 1 - n);  // R[off + i] = s[n - i]
    uint64_t acc = 0;
    for (int w = 0; w <= L / 64; ++w) acc ^= Cp[w] & window(off + 64ull * w);
    // C has no bits above degree L, so the words up to L / 64 hold the whole sum
    const int d = __builtin_parityll(acc);
    if (!d) {
      ++m;
      continue;
    }
    const bool grow = 2 * L <= n;
    if (grow) T = Cp;
    const int ws = m >> 6, bs = m & 63;
    for (int q = W + 1; q >= 0; --q) {
      const uint64_t lo = q - ws >= 0 ? Bp[q - ws] << bs : 0;
      const uint64_t hi = (bs && q - ws - 1 >= 0) ? Bp[q - ws - 1] >> (64 - bs) : 0;
      Cp[q] ^= lo | hi;
    }
    if (grow) {
      L = n + 1 - L;
      Bp = T;
      m = 1;
    } else {
      ++m;
    }
  }
  if (L != kDeg) {
    J.error = "Berlekamp-Massey found a recurrence of degree " + std::to_string(L) + ", not 19937";
    return false;
  }
  // phi(x) = x^L C(1/x): coefficient j of phi is C_{L - j}
  std::vector<uint64_t> phi(kPW + 1, 0);
  for (int j = 0; j <= kDeg; ++j)
    if (bit(Cp, (uint64_t)(kDeg - j))) phi[j >> 6] |= 1ull << (j & 63);
  J.phish.assign((size_t)64 * (kPW + 1), 0);
  for (int s2 = 0; s2 < 64; ++s2)
    for (int q = 0; q <= kPW; ++q) {
      const uint64_t lo = phi[q] << s2;
      const uint64_t hi = (q > 0 && s2) ? phi[q - 1] >> (64 - s2) : 0;
      J.phish[(size_t)s2 * (kPW + 1) + q] = lo | hi;
    }
  return true;
}

// P_0 = 1 and P_1 = x^W mod phi of a substream length W
void start_set(JumpTable& J, uint64_t W, JumpSet& S) {
  std::vector<uint64_t> one(kPW, 0), x1(kPW, 0);
  one[0] = 1;
  x1[0] = 2;
  S.polys.push_back(one);
  S.polys.push_back(powmod(x1, W, J.phish));
}

// the jump polynomials of substreams 0 .. blocks-1 of length W on `device` (host work once per
// process and W)
const DevPositions* jump_polys(uint64_t W, uint64_t blocks, int device, const char** err) {
  JumpTable& J = jump_table();
  std::lock_guard<std::mutex> lock(J.mu);
  if (!J.ready) {
    if (!build_phi(J)) {
      *err = J.error.c_str();
      return nullptr;
    }
    J.ready = true;
  }
  JumpSet& S = J.sets[W];
  if (S.polys.empty()) start_set(J, W, S);
  if (S.polys.size() < blocks) {
    const uint64_t have = S.polys.size();
    S.polys.resize(blocks);
    const unsigned nt = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
    const uint64_t per = (blocks - have + nt - 1) / nt;
    std::vector<std::thread> th;
    for (unsigned t = 0; t < nt; ++t) {
      const uint64_t lo = have + t * per, hi = std::min<uint64_t>(blocks, lo + per);
      if (lo >= hi) break;
      th.emplace_back([&J, &S, lo, hi] {
        std::vector<uint64_t> cur = powmod(S.polys[1], lo, J.phish);
        for (uint64_t b = lo; b < hi; ++b) {
          S.polys[b] = cur;
          if (b + 1 < hi) cur = mulmod(cur, S.polys[1], J.phish);
        }
      });
    }
    for (auto& x : th) x.join();
  }
  auto& d = S.dev[device];
  if (d.blocks < blocks) {  // the old copy is kept: kernels in flight may still read it
    std::vector<uint16_t> pos;
    std::vector<uint32_t> off(blocks + 1);
    for (uint64_t b = 0; b < blocks; ++b) {
      off[b] = (uint32_t)pos.size();
      const std::vector<uint64_t>& P = S.polys[b];
      for (int i = 0; i < kDeg; ++i)
        if ((P[i >> 6] >> (i & 63)) & 1u) pos.push_back((uint16_t)i);
      while ((pos.size() - off[b]) % 4) pos.push_back(kZeroPos);
    }
    off[blocks] = (uint32_t)pos.size();
    DevPositions nd;
    if (cudaMalloc(&nd.pos, pos.size() * 2 + 8) != cudaSuccess || cudaMalloc(&nd.off, off.size() * 4) != cudaSuccess) {
      *err = "cudaMalloc of the jump polynomials failed";
      return nullptr;
    }
    cudaMemcpy(nd.pos, pos.data(), pos.size() * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(nd.off, off.data(), off.size() * 4, cudaMemcpyHostToDevice);
    nd.blocks = blocks;
    d = nd;
  }
  return &d;
}

// first[t] / second[t]: the two smallest iterations that targeted position t, in one pass.  The
// atomicMin on first returns what it displaced: every iteration but the smallest is displaced or
// loses at some point, and the loser of each exchange (the larger of the two) goes to second, so
// second ends as the smallest of all but the first (iterations are distinct)
__global__ void touch_pass(const uint32_t* __restrict__ draws, uint64_t len, uint64_t ndraws,
                           uint32_t* __restrict__ first, uint32_t* __restrict__ second) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t d = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; d < ndraws; d += stride) {
    const uint32_t tgt = draws[d];
    const uint32_t it = (uint32_t)(len - d);
    const uint32_t old = atomicMin(&first[tgt], it);
    if (old != kNone) atomicMin(&second[tgt], old > it ? old : it);
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

// CPU check of the jump-ahead (tests): the window of substream b computed by the correlation
// with P_b against the engine advanced output by output; 0 when every word agrees (the first
// word up to its 31 low bits, which the twist never reads) and the next 312 outputs match
int mt_jump_check(uint64_t engine_seed, uint64_t b, const char** err) {
  constexpr uint64_t W = 312ull * 128ull;
  JumpTable& J = jump_table();
  std::vector<uint64_t> P;
  {
    std::lock_guard<std::mutex> lock(J.mu);
    if (!J.ready) {
      if (!build_phi(J)) {
        *err = J.error.c_str();
        return -1;
      }
      J.ready = true;
    }
    JumpSet& S = J.sets[W];
    if (S.polys.empty()) start_set(J, W, S);
    for (uint64_t q = S.polys.size(); q <= b; ++q) S.polys.push_back(mulmod(S.polys[q - 1], S.polys[1], J.phish));
    P = S.polys[b];
  }
  const uint64_t total = b * W + 2 * kMtN + kMtSeqWords;
  std::vector<uint64_t> x(total);
  uint64_t v = engine_seed;
  x[0] = v;
  for (int i = 1; i < kMtN; ++i) {
    v = 6364136223846793005ULL * (v ^ (v >> 62)) + (uint64_t)i;
    x[i] = v;
  }
  for (uint64_t k = kMtN; k < total; ++k) x[k] = twist_word(x[k - kMtN], x[k - kMtN + 1], x[k - kMtN + 156]);
  std::vector<uint64_t> w(kMtN, 0);
  for (int i = 0; i < kDeg; ++i)
    if ((P[i >> 6] >> (i & 63)) & 1u)
      for (int j = 0; j < kMtN; ++j) w[j] ^= x[i + j];
  const uint64_t base = b * W;
  if ((w[0] ^ x[base]) & 0xFFFFFFFF80000000ULL) return 1;
  for (int j = 1; j < kMtN; ++j)
    if (w[j] != x[base + j]) return 2;
  std::vector<uint64_t> ext(w);  // the next twist from the computed window
  for (int k = 0; k < kMtN; ++k) ext.push_back(twist_word(ext[k], ext[k + 1], ext[k + 156]));
  for (int k = 0; k < kMtN; ++k)
    if (temper(ext[kMtN + k]) != temper(x[base + kMtN + k])) return 3;
  return 0;
}

int launch_random_indices(uint64_t engine_seed, uint64_t len, uint64_t count, const RandomScratch& s,
                          cudaStream_t stream, const char** err) {
  const uint64_t words = (len + 31) / 32;
  cudaMemsetAsync(s.bitmap, 0, words * sizeof(uint32_t), stream);
  if (count >= len) {
    count_launches(4);
    fill_prefix<<<sm_grid(words, 256), 256, 0, stream>>>(s.bitmap, len);
  } else {
    const uint64_t ndraws = len - count;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    // substreams: one wave of CTAs, kSubPerCta each, W outputs per substream (a multiple of 312)
    const uint64_t want = (uint64_t)sms * kSubPerCta;
    const uint64_t W = ((ndraws + want * kMtN - 1) / (want * kMtN)) * kMtN;
    const uint64_t nsub = (ndraws + W - 1) / W;
    if (nsub > s.mt_blocks_cap) {
      *err = "substream windows scratch too small";
      return DMB_CUDA;
    }
    const DevPositions* jp = jump_polys(W, nsub, dev, err);
    if (!jp) return DMB_CUDA;
    count_launches(8);
    // DMB_MT_FORCE_FIXUP=1 (tests): report a rejection at output 0, so the sequential replay
    // rewrites every draw -- it must reproduce the substreams' draws exactly
    const char* ff = std::getenv("DMB_MT_FORCE_FIXUP");
    cudaMemsetAsync(s.mt_reject, (ff && ff[0] == '1') ? 0x00 : 0xff, sizeof(unsigned long long), stream);
    mt_seq_kernel<<<1, kMtThreads, 0, stream>>>(engine_seed, s.mt_seq);
    const int smem = (int)((kMtSeqWords + 4 * kMtN) * 8);
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(mt_block_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      attr = true;
    }
    const unsigned ctas = (unsigned)((nsub + kSubPerCta - 1) / kSubPerCta);
    mt_block_kernel<<<ctas, kBlockThreads, smem, stream>>>(s.mt_seq, jp->pos, jp->off, W, nsub, len, ndraws,
                                                           s.draws, s.mt_windows, s.mt_reject);
    mt_fixup_kernel<<<1, kMtThreads, 0, stream>>>(s.mt_windows, W, len, ndraws, s.draws, s.mt_reject);
    cudaMemsetAsync(s.first, 0xff, len * sizeof(uint32_t), stream);
    cudaMemsetAsync(s.second, 0xff, len * sizeof(uint32_t), stream);
    touch_pass<<<sm_grid(ndraws, 256), 256, 0, stream>>>(s.draws, len, ndraws, s.first, s.second);
    resolve_kernel<<<sm_grid(count, 256), 256, 0, stream>>>(count, s.first, s.second, s.bitmap);
  }
  const uint64_t blocks = (words + kScanBlock - 1) / kScanBlock;
  uint32_t* partial = s.rank + words + 1;  // scratch tail of the rank array
  block_popc<<<(unsigned)blocks, kScanBlock, 0, stream>>>(s.bitmap, words, partial);
  scan_partials<<<1, kScanBlock, 0, stream>>>(partial, blocks);
  word_ranks<<<(unsigned)blocks, kScanBlock, 0, stream>>>(s.bitmap, words, partial, s.rank, s.idx);
  return DMB_OK;
}

}  // namespace dmb
