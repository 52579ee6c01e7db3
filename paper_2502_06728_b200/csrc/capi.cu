// capi.cu -- the extern "C" boundary (include/demo_b200.h) and the host runtime
// around the kernels: per-device context (basis tables, status latch, Random
// index scratch), reference-exact validation (the ConfigError / ProtocolError
// rules of replicate.cpp and optim.cpp), step scalars computed in double on the
// host (std::pow bias corrections, optim.cpp:62-63), and dispatch by scheme.
#include <atomic>
#include <cstdarg>
#include <cmath>
#include <cstdio>
#include <mutex>
#include <tuple>
#include <vector>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "dmb_internal.cuh"

namespace dmb {
static std::atomic<uint64_t> g_launches{0};
void count_launches(int n) { g_launches.fetch_add((uint64_t)n, std::memory_order_relaxed); }
static std::atomic<int> g_sm_reserve{0};
int sm_reserve() { return g_sm_reserve.load(std::memory_order_relaxed); }

namespace {
std::mutex g_timer_mu;
bool g_timer_on = false;
std::vector<std::pair<cudaEvent_t, cudaEvent_t>> g_timer_pairs;  // recorded, not yet read
std::vector<std::pair<cudaEvent_t, cudaEvent_t>> g_timer_pool;   // read, reusable
cudaEvent_t g_timer_open = nullptr;
}  // namespace
void timer_begin(cudaStream_t stream) {
  std::lock_guard<std::mutex> l(g_timer_mu);
  if (!g_timer_on) return;
  cudaEvent_t b = nullptr, e = nullptr;
  if (!g_timer_pool.empty()) {
    std::tie(b, e) = g_timer_pool.back();
    g_timer_pool.pop_back();
  } else {
    cudaEventCreate(&b);
    cudaEventCreate(&e);
  }
  cudaEventRecord(b, stream);
  g_timer_pairs.emplace_back(b, e);
  g_timer_open = e;
}
void timer_end(cudaStream_t stream) {
  std::lock_guard<std::mutex> l(g_timer_mu);
  if (!g_timer_on || !g_timer_open) return;
  cudaEventRecord(g_timer_open, stream);
  g_timer_open = nullptr;
}
}  // namespace dmb

namespace dmb {
__global__ void latch_export_kernel(const DevStatus* st, int32_t* flag) {
  *flag = st->first_bad != kNoBad ? 1 : 0;
}
__global__ void latch_import_kernel(DevStatus* st, const int32_t* flag) {
  if (*flag && st->first_bad == kNoBad) st->first_bad = kNoBad - 1ull;  // kPeerBad
}
}  // namespace dmb

using namespace dmb;

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define DMB_CUDA_TRY(expr)                                                             \
  do {                                                                                 \
    cudaError_t e_ = (expr);                                                           \
    if (e_ != cudaSuccess) return fail(DMB_CUDA, "%s: %s", #expr, cudaGetErrorString(e_)); \
  } while (0)

int last_launch() {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(DMB_CUDA, "kernel launch: %s", cudaGetErrorString(e));
  return DMB_OK;
}

constexpr double kPi = 3.14159265358979323846264338327950288;

// DctPlan basis, transform.cpp:41-54: same expression order and libm cos as the
// reference, so the FP64 table is bit-identical to the oracle's.
std::vector<double> host_basis(int s) {
  std::vector<double> b((size_t)s * s);
  const double n = (double)s;
  const double c0 = std::sqrt(1.0 / n);
  const double cj = std::sqrt(2.0 / n);
  for (int j = 0; j < s; ++j) {
    const double scale = j == 0 ? c0 : cj;
    for (int i = 0; i < s; ++i)
      b[(size_t)j * s + i] = scale * std::cos(kPi * (2.0 * (double)i + 1.0) * (double)j / (2.0 * n));
  }
  return b;
}

struct BasisBuf {
  float* B = nullptr;
  float* BT = nullptr;
  double* B64 = nullptr;  // B64 | B64T, each s*s
  float* tf32 = nullptr;  // Bhi | Blo | BThi | BTlo, each s*s
};

// round to TF32 (10 explicit mantissa bits), nearest, ties away: cvt.rna.tf32.f32
float tf32_rna_host(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  if ((u & 0x7f800000u) != 0x7f800000u) u = (u + 0x1000u) & 0xffffe000u;
  std::memcpy(&f, &u, 4);
  return f;
}

struct RandomKey {
  uint64_t seed = 0, step = 0, len = 0, count = 0;
  uint32_t shard = 0;
  bool valid = false;
  bool operator==(const RandomKey& o) const {
    return valid && o.valid && seed == o.seed && step == o.step && len == o.len &&
           count == o.count && shard == o.shard;
  }
};

}  // namespace

struct dmb_ctx {
  int device = 0;
  DevStatus* status = nullptr;  // step latch: prepare/apply/step paths
  DevStatus* aux = nullptr;     // standalone select_and_encode / decode_and_merge
  std::map<int, BasisBuf> bases;
  RandomScratch rnd{};
  RandomKey rnd_key;
  uint64_t rnd_len_cap = 0;
  uint32_t* fb_list = nullptr;  // chunks the tensor-core path hands to the FP64 kernel
  unsigned* fb_count = nullptr;
  uint64_t fb_cap = 0;
  int wire_format = DMB_WIRE_REFERENCE;  // DeMo exchange layout of the updates encoded here
  uint8_t* scratch = nullptr;             // extract_fast_components' payload body
  uint64_t scratch_cap = 0;
};

namespace {

int get_basis(dmb_ctx* ctx, int s, Basis* out) {
  auto it = ctx->bases.find(s);
  if (it == ctx->bases.end()) {
    const std::vector<double> b64 = host_basis(s);
    std::vector<float> b((size_t)s * s), bt((size_t)s * s);
    for (int j = 0; j < s; ++j)
      for (int i = 0; i < s; ++i) {
        b[(size_t)j * s + i] = (float)b64[(size_t)j * s + i];
        bt[(size_t)i * s + j] = (float)b64[(size_t)j * s + i];
      }
    std::vector<float> split((size_t)4 * s * s);
    for (int j = 0; j < s; ++j)
      for (int i = 0; i < s; ++i) {
        const double v = b64[(size_t)j * s + i];
        const float hi = tf32_rna_host((float)v);
        const float lo = tf32_rna_host((float)(v - (double)hi));
        split[(size_t)j * s + i] = hi;                      // Bhi[j][i]
        split[(size_t)s * s + (size_t)j * s + i] = lo;      // Blo[j][i]
        split[(size_t)2 * s * s + (size_t)i * s + j] = hi;  // BThi[i][j]
        split[(size_t)3 * s * s + (size_t)i * s + j] = lo;  // BTlo[i][j]
      }
    BasisBuf buf;
    DMB_CUDA_TRY(cudaMalloc(&buf.tf32, split.size() * sizeof(float)));
    DMB_CUDA_TRY(cudaMemcpy(buf.tf32, split.data(), split.size() * sizeof(float), cudaMemcpyHostToDevice));
    DMB_CUDA_TRY(cudaMalloc(&buf.B, b.size() * sizeof(float)));
    DMB_CUDA_TRY(cudaMalloc(&buf.BT, bt.size() * sizeof(float)));
    DMB_CUDA_TRY(cudaMalloc(&buf.B64, 2 * b64.size() * sizeof(double)));
    std::vector<double> b64t((size_t)s * s);
    for (int j = 0; j < s; ++j)
      for (int i = 0; i < s; ++i) b64t[(size_t)i * s + j] = b64[(size_t)j * s + i];
    DMB_CUDA_TRY(cudaMemcpy(buf.B64 + b64.size(), b64t.data(), b64t.size() * sizeof(double), cudaMemcpyHostToDevice));
    DMB_CUDA_TRY(cudaMemcpy(buf.B, b.data(), b.size() * sizeof(float), cudaMemcpyHostToDevice));
    DMB_CUDA_TRY(cudaMemcpy(buf.BT, bt.data(), bt.size() * sizeof(float), cudaMemcpyHostToDevice));
    DMB_CUDA_TRY(cudaMemcpy(buf.B64, b64.data(), b64.size() * sizeof(double), cudaMemcpyHostToDevice));
    it = ctx->bases.emplace(s, buf).first;
  }
  out->s = s;
  out->B = it->second.B;
  out->BT = it->second.BT;
  out->B64 = it->second.B64;
  const size_t ss = (size_t)s * s;
  out->B64T = it->second.B64 + ss;
  out->Bhi = it->second.tf32;
  out->Blo = it->second.tf32 + ss;
  out->BThi = it->second.tf32 + 2 * ss;
  out->BTlo = it->second.tf32 + 3 * ss;
  return DMB_OK;
}

unsigned long long* g_dbg = nullptr;  // event timestamps of the next tc3 launch (tuning)

// fallback-list scratch for the tensor-core path (one slot per chunk)
int attach_fallback(dmb_ctx* ctx, ChunkArgs* a) {
  a->dbg = g_dbg;
  if (a->geo.nchunks > ctx->fb_cap) {
    cudaFree(ctx->fb_list);
    DMB_CUDA_TRY(cudaMalloc(&ctx->fb_list, (a->geo.nchunks + 1) * sizeof(uint32_t)));
    ctx->fb_cap = a->geo.nchunks;
  }
  if (!ctx->fb_count) DMB_CUDA_TRY(cudaMalloc(&ctx->fb_count, sizeof(unsigned)));
  a->fb_list = ctx->fb_list;
  a->fb_count = ctx->fb_count;
  return DMB_OK;
}

uint64_t value_bits(int32_t d) { return d == DMB_FP16 ? 16 : (d == DMB_TERNARY ? 2 : 32); }

uint64_t wire_bytes(uint64_t nv, uint64_t ni, int32_t d) {
  return (nv * value_bits(d) + ni * 32 + 7) / 8;  // replicate.cpp:44-48
}

uint64_t period_of(double c) {
  const long long p = std::llround(1.0 / c);  // replicate.cpp:50-53
  return p < 1 ? 1 : (uint64_t)p;
}

// selection_count, replicate.cpp:146-156
int selection_count(double c, uint64_t len, uint64_t* out) {
  const long long n = std::llround(c * (double)len);
  if (n < 1)
    return fail(DMB_CONFIG, "compression %g selects no components from a vector of length %llu", c,
                (unsigned long long)len);
  *out = (uint64_t)n < len ? (uint64_t)n : len;
  return DMB_OK;
}

int validate_dtype(const dmb_rep_cfg* cfg) {
  if (cfg->transfer_dtype < DMB_FP32 || cfg->transfer_dtype > DMB_TERNARY)
    return fail(DMB_CONFIG, "unknown transfer dtype %d", cfg->transfer_dtype);
  return DMB_OK;
}

// The header select_and_encode produces (replicate.cpp:187-237).
int plan(const dmb_rep_cfg* cfg, uint64_t len, uint64_t step, uint32_t shard, dmb_update* u) {
  if (int rc = validate_dtype(cfg)) return rc;
  void* body = u->body;
  std::memset(u, 0, sizeof *u);
  u->body = body;
  u->scheme = cfg->scheme;
  u->step = step;
  u->shard_id = shard;
  u->length = len;
  switch (cfg->scheme) {
    case DMB_FULL:
      u->n_values = len;
      break;
    case DMB_DILOCO:
      if (step % period_of(cfg->compression) != 0) u->empty = 1;
      else u->n_values = len;
      break;
    case DMB_RANDOM: {
      uint64_t n = 0;
      if (int rc = selection_count(cfg->compression, len, &n)) return rc;
      u->n_values = n;
      break;
    }
    case DMB_STRIDING: {
      const uint64_t n = period_of(cfg->compression);
      if (n > len)  // replicate.cpp:176-180
        return fail(DMB_CONFIG, "stride period %llu exceeds vector length %llu",
                    (unsigned long long)n, (unsigned long long)len);
      const uint64_t off = step % n;
      u->n_values = off >= len ? 0 : (len - off + n - 1) / n;
      break;
    }
    case DMB_DEMO: {
      if (cfg->chunk_size == 0) return fail(DMB_CONFIG, "chunk size must be positive");
      if (cfg->top_k == 0 || cfg->top_k > cfg->chunk_size)  // transform.cpp:96-101
        return fail(DMB_CONFIG, "top_k %llu out of range for chunk size %llu",
                    (unsigned long long)cfg->top_k, (unsigned long long)cfg->chunk_size);
      if (cfg->chunk_size > 256)
        return fail(DMB_CONFIG, "chunk size %llu above the device limit 256",
                    (unsigned long long)cfg->chunk_size);
      const uint64_t nc = (len + cfg->chunk_size - 1) / cfg->chunk_size;
      u->chunk_size = cfg->chunk_size;
      u->top_k = cfg->top_k;
      u->n_values = nc * cfg->top_k;
      u->n_indices = u->n_values;
      break;
    }
    default:
      return fail(DMB_CONFIG, "unknown replication scheme %d", cfg->scheme);
  }
  if (len >= (1ull << 32) && (cfg->scheme == DMB_RANDOM || cfg->scheme == DMB_STRIDING))
    return fail(DMB_CONFIG, "index sets are uint32 (replicate.cpp:162): length %llu too long",
                (unsigned long long)len);
  u->bytes = wire_bytes(u->n_values, u->n_indices, cfg->transfer_dtype);
  return DMB_OK;
}

uint64_t capacity(const dmb_rep_cfg* cfg, uint64_t len) {
  uint64_t nv = len, ni = 0;
  if (cfg->scheme == DMB_DEMO && cfg->chunk_size) {
    nv = ((len + cfg->chunk_size - 1) / cfg->chunk_size) * cfg->top_k;
    ni = nv;
  }
  return ((wire_bytes(nv, ni, cfg->transfer_dtype) + 15) / 16) * 16 + 16;
}

float half_to_float(uint16_t h) {
  __half_raw r;
  r.x = h;
  return __half2float(__half(r));
}
uint16_t float_to_half(float v) {
  const __half_raw r = __float2half_rn(v);
  return r.x;
}

bool is_mask(const dmb_update* u) { return u->scheme == DMB_DEMO && u->wire_format != DMB_WIRE_REFERENCE; }
uint64_t chunks_of(const dmb_update* u) { return u->chunk_size ? (u->length + u->chunk_size - 1) / u->chunk_size : 0; }
// dtype of the packed values actually in the body
int32_t body_value_dtype(const dmb_update* u, int32_t dtype) {
  return u->wire_format == DMB_WIRE_MASK_SIGN ? DMB_TERNARY : dtype;
}
uint64_t mask_body_bytes(const dmb_update* u, int32_t dtype) {
  if (u->wire_format == DMB_WIRE_MASK_SIGN) return 24 * chunks_of(u);  // masks + codes by column
  return 8 * chunks_of(u) + (u->n_values * value_bits(body_value_dtype(u, dtype)) + 7) / 8;
}

uint8_t* values_region(const dmb_update* u) {
  if (is_mask(u)) return static_cast<uint8_t*>(u->body) + 8 * chunks_of(u);
  return static_cast<uint8_t*>(u->body) + u->n_indices * 4;
}

int prep_values_region(const dmb_update* u, int32_t dtype, cudaStream_t st) {
  dtype = body_value_dtype(u, dtype);
  if (dtype == DMB_TERNARY && u->n_values) {
    const uint64_t vb = (u->n_values * 2 + 7) / 8;
    DMB_CUDA_TRY(cudaMemsetAsync(values_region(u), 0, ((vb + 3) / 4) * 4, st));
  }
  return DMB_OK;
}

DemoGeometry geometry(const dmb_rep_cfg* cfg, uint64_t len) {
  DemoGeometry g{};
  g.len = len;
  g.s = (int)cfg->chunk_size;
  g.k = (int)cfg->top_k;
  g.nchunks = (len + g.s - 1) / g.s;
  g.dtype = cfg->transfer_dtype;
  g.sign_mode = cfg->sign_mode != 0;
  return g;
}

// The device index set of a Random (step, shard): generated once and reused by
// encode and merge of the same step (the reference re-derives it twice).
int ensure_random(dmb_ctx* ctx, const dmb_rep_cfg* cfg, uint64_t step, uint32_t shard,
                  uint64_t len, uint64_t count, cudaStream_t st) {
  RandomKey key;
  key.seed = cfg->seed;
  key.step = step;
  key.len = len;
  key.count = count;
  key.shard = shard;
  key.valid = true;
  if (key == ctx->rnd_key) return DMB_OK;
  if (len > ctx->rnd_len_cap) {
    RandomScratch& r = ctx->rnd;
    cudaFree(r.draws);
    cudaFree(r.first);
    cudaFree(r.second);
    cudaFree(r.bitmap);
    cudaFree(r.rank);
    cudaFree(r.idx);
    const uint64_t words = (len + 31) / 32;
    DMB_CUDA_TRY(cudaMalloc(&r.draws, len * 4 + 4));
    DMB_CUDA_TRY(cudaMalloc(&r.first, len * 4 + 4));
    DMB_CUDA_TRY(cudaMalloc(&r.second, len * 4 + 4));
    DMB_CUDA_TRY(cudaMalloc(&r.bitmap, words * 4 + 4));
    DMB_CUDA_TRY(cudaMalloc(&r.rank, (words + 1 + words / 1024 + 2) * 4));
    DMB_CUDA_TRY(cudaMalloc(&r.idx, len * 4 + 4));
    r.capacity = len;
    ctx->rnd_len_cap = len;
  }
  RandomScratch& r = ctx->rnd;
  const uint64_t blocks = kMtMaxSubstreams;
  if (!r.mt_seq) {
    DMB_CUDA_TRY(cudaMalloc(&r.mt_seq, kMtSeqWords * 8));
    DMB_CUDA_TRY(cudaMalloc(&r.mt_reject, sizeof(unsigned long long)));
  }
  if (blocks > r.mt_blocks_cap) {
    cudaFree(r.mt_windows);
    DMB_CUDA_TRY(cudaMalloc(&r.mt_windows, blocks * 312 * 8));
    r.mt_blocks_cap = blocks;
  }
  // Rng(mix_seed(seed, step, shard)) seeds the engine with mix_seed(.) once more
  // (rng.hpp:21, replicate.cpp:167).
  auto mix64 = [](uint64_t z) {
    z += 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
  };
  const uint64_t derived = mix64(mix64(mix64(cfg->seed) ^ step) ^ (uint64_t)shard);
  const char* err = nullptr;
  if (launch_random_indices(mix64(derived), len, count, ctx->rnd, st, &err) != DMB_OK)
    return fail(DMB_CUDA, "random index set: %s", err ? err : "?");
  if (int rc = last_launch()) return rc;
  ctx->rnd_key = key;
  return DMB_OK;
}

int sparse_sel(dmb_ctx* ctx, const dmb_rep_cfg* cfg, const dmb_update* u, SparseSel* sel,
               cudaStream_t st) {
  std::memset(sel, 0, sizeof *sel);
  sel->len = u->length;
  sel->count = u->n_values;
  sel->scheme = u->empty ? 0 : cfg->scheme;
  if (cfg->scheme == DMB_STRIDING) {
    sel->period = period_of(cfg->compression);
    sel->offset = u->step % sel->period;
  } else if (cfg->scheme == DMB_RANDOM) {
    if (int rc = ensure_random(ctx, cfg, u->step, u->shard_id, u->length, u->n_values, st)) return rc;
    sel->bitmap = ctx->rnd.bitmap;
    sel->rank = ctx->rnd.rank;
  }
  return DMB_OK;
}

SgdScalars sgd_scalars(double beta, double lr) {
  SgdScalars s;
  s.beta = (float)beta;
  s.lr = (float)lr;
  return s;
}

// optim.cpp:60-63: steps += 1; bias corrections with std::pow in double
AdamScalars adam_scalars(const dmb_opt_cfg* o, uint64_t steps_after, double lr) {
  AdamScalars a{};
  const double bc1 = 1.0 - std::pow(o->adam_beta1, (double)steps_after);
  const double bc2 = 1.0 - std::pow(o->adam_beta2, (double)steps_after);
  a.beta1 = (float)o->adam_beta1;
  a.one_minus_beta1 = (float)(1.0 - o->adam_beta1);
  a.beta2 = (float)o->adam_beta2;
  a.one_minus_beta2 = (float)(1.0 - o->adam_beta2);
  a.inv_bc1 = (float)(1.0 / bc1);
  a.inv_bc2 = (float)(1.0 / bc2);
  a.eps = (float)o->adam_eps;
  a.lr = (float)lr;
  a.lr_bc1 = (float)(lr / bc1);
  a.lr_wd = o->weight_decay != 0.0 ? (float)(lr * o->weight_decay) : 0.0f;
  return a;
}

// decode_and_merge validation, replicate.cpp:241-253, :263, :273-275, :284-293
int validate_updates(const dmb_update* ups, uint64_t n, const dmb_rep_cfg* cfg) {
  if (n == 0 || !ups) return fail(DMB_PROTOCOL, "decode_and_merge needs at least one update");
  if (n > (uint64_t)kMaxReplicas) return fail(DMB_PROTOCOL, "at most %d replicas per merge", kMaxReplicas);
  const dmb_update& r = ups[0];
  if (r.scheme != cfg->scheme) return fail(DMB_PROTOCOL, "update scheme does not match the config");
  for (uint64_t i = 0; i < n; ++i) {
    const dmb_update& u = ups[i];
    if (u.scheme != r.scheme || u.step != r.step || u.shard_id != r.shard_id || u.length != r.length)
      return fail(DMB_PROTOCOL, "replicas disagree on scheme, step, shard or length");
    if (u.empty) return fail(DMB_PROTOCOL, "cannot merge an update with no payload");
    if (u.n_values != r.n_values) return fail(DMB_PROTOCOL, "replicas disagree on transmitted value count");
    if (!u.body && u.n_values) return fail(DMB_PROTOCOL, "update has no device body");
  }
  switch (cfg->scheme) {
    case DMB_FULL:
    case DMB_DILOCO:
      if (r.n_values != r.length) return fail(DMB_PROTOCOL, "full update has the wrong length");
      break;
    case DMB_RANDOM:
    case DMB_STRIDING: {
      dmb_update expect{};
      if (int rc = plan(cfg, r.length, r.step, r.shard_id, &expect)) return rc;
      if (expect.n_values != r.n_values)
        return fail(DMB_PROTOCOL, "selected value count does not match the derived index set");
      break;
    }
    case DMB_DEMO: {
      if (r.chunk_size != cfg->chunk_size || r.top_k != cfg->top_k)
        return fail(DMB_PROTOCOL, "chunk geometry does not match the config");
      for (uint64_t i = 0; i < n; ++i)
        if (ups[i].wire_format != r.wire_format)
          return fail(DMB_PROTOCOL, "updates of one merge use different wire formats");
      const uint64_t expected = ((r.length + cfg->chunk_size - 1) / cfg->chunk_size) * cfg->top_k;
      for (uint64_t i = 0; i < n; ++i)
        if (ups[i].n_indices != expected || ups[i].n_values != expected)
          return fail(DMB_PROTOCOL, "frequency payload does not match the chunk layout");
      break;
    }
    default:
      return fail(DMB_CONFIG, "unknown replication scheme %d", cfg->scheme);
  }
  return DMB_OK;
}

Bodies bodies_of(const dmb_update* ups, uint64_t n, bool values_only) {
  Bodies b{};
  b.R = (int)n;
  for (uint64_t i = 0; i < n; ++i)
    b.body[i] = values_only ? values_region(&ups[i]) : static_cast<const uint8_t*>(ups[i].body);
  return b;
}

int clear_aux(dmb_ctx* ctx, cudaStream_t st) {
  DMB_CUDA_TRY(cudaMemsetAsync(&ctx->aux->first_bad, 0xff, sizeof(unsigned long long), st));
  DMB_CUDA_TRY(cudaMemsetAsync(&ctx->aux->protocol_error, 0, sizeof(unsigned int), st));
  return DMB_OK;
}

int check_aux_protocol(dmb_ctx* ctx, cudaStream_t st) {
  unsigned int perr = 0;
  DMB_CUDA_TRY(cudaMemcpyAsync(&perr, &ctx->aux->protocol_error, sizeof perr, cudaMemcpyDeviceToHost, st));
  DMB_CUDA_TRY(cudaStreamSynchronize(st));
  if (perr) return fail(DMB_PROTOCOL, "frequency index out of range");
  return DMB_OK;
}

// The DeMo exchange layout this context emits for a vector of `len`: MASK wherever the
// tensor-core encoder can run (s = 64, whole chunks, tensor maps available), decided from the
// configuration alone so a caller can size its exchange slots with dmb_plan_exchange; the
// encoder then fails loudly instead of changing layout (e.g. for misaligned vectors).
bool mask_layout(const dmb_ctx* ctx, const dmb_rep_cfg* cfg, uint64_t len) {
  return ctx->wire_format != DMB_WIRE_REFERENCE && cfg->scheme == DMB_DEMO && cfg->chunk_size == 64 && len >= 64 &&
         len % 64 == 0 && tc_enabled() && tc3_available();
}
void set_mask_header(const dmb_rep_cfg* cfg, dmb_update* out) {
  out->wire_format = (cfg->sign_mode || cfg->transfer_dtype == DMB_TERNARY) ? DMB_WIRE_MASK_SIGN : DMB_WIRE_MASK;
  out->bytes = mask_body_bytes(out, cfg->transfer_dtype);
}

// Encode one vector (v = g, or m_acc from beta*m_in + g when sgd) into *out.
int encode(dmb_ctx* ctx, DevStatus* st, bool sgd, const float* g, const float* m_in, float* m_out,
           double beta, uint64_t len, const dmb_rep_cfg* cfg, uint64_t step, uint32_t shard,
           dmb_update* out, float* local_q, float* m_accum, cudaStream_t s,
           const float* const* srcs = nullptr, int n_src = 0) {
  if (!out) return fail(DMB_CONFIG, "update output is NULL");
  if (int rc = plan(cfg, len, step, shard, out)) return rc;
  if (!out->body && out->n_values) return fail(DMB_CONFIG, "update body is NULL");
  if (len == 0) return DMB_OK;
  if (cfg->scheme == DMB_DEMO) {
    ChunkArgs a{};
    a.geo = geometry(cfg, len);
    if (int rc = get_basis(ctx, a.geo.s, &a.basis)) return rc;
    a.g = g;
    a.m_in = m_in;
    a.m_out = m_out;
    a.local_q = local_q;
    a.m_accum = m_accum;
    a.body = static_cast<uint8_t*>(out->body);
    a.sgd = sgd_scalars(beta, 0.0);
    a.status = st;
    a.n_src = n_src;
    for (int q = 0; q < n_src; ++q) a.g_src[q] = srcs[q];
    if (int rc = attach_fallback(ctx, &a)) return rc;
    if (mask_layout(ctx, cfg, len)) {
      if (!tc3_supported(sgd ? ChunkMode::EncodeSgd : ChunkMode::EncodeAdam, a))
        return fail(DMB_CONFIG, "the MASK exchange layout needs the tensor-core encoder: 16-byte aligned vectors%s "
                    "and no local_q / m_accum output", sgd ? " (distinct momentum buffers allowed)" : "");
      set_mask_header(cfg, out);
      a.geo.wire_mask = 1;
    }
    if (int rc = prep_values_region(out, cfg->transfer_dtype, s)) return rc;
    launch_chunk_kernel(sgd ? ChunkMode::EncodeSgd : ChunkMode::EncodeAdam, a, s);
    return last_launch();
  }
  if (int rc = prep_values_region(out, cfg->transfer_dtype, s)) return rc;
  SparseSel sel;
  if (int rc = sparse_sel(ctx, cfg, out, &sel, s)) return rc;
  launch_sparse_encode(sel, sgd, g, m_in, m_out, (float)beta, local_q, m_accum,
                       out->n_values ? values_region(out) : nullptr, cfg->transfer_dtype,
                       cfg->sign_mode != 0, st, s);
  return last_launch();
}

cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

// first_bad of a step failed on another rank of the group (dmb_latch_import)
constexpr unsigned long long kPeerBad = kNoBad - 1ull;

}  // namespace

extern "C" {

int dmb_abi_version(void) { return DMB_ABI_VERSION; }
const char* dmb_last_error(void) { return g_err.c_str(); }

int dmb_ctx_create(int device, dmb_ctx** out) {
  if (!out) return fail(DMB_CONFIG, "ctx output is NULL");
  DMB_CUDA_TRY(cudaSetDevice(device));
  std::unique_ptr<dmb_ctx> ctx(new dmb_ctx());
  ctx->device = device;
  DMB_CUDA_TRY(cudaMalloc(&ctx->status, sizeof(DevStatus)));
  DMB_CUDA_TRY(cudaMalloc(&ctx->aux, sizeof(DevStatus)));
  DevStatus clean{kNoBad, 0, 0, 0};
  DMB_CUDA_TRY(cudaMemcpy(ctx->status, &clean, sizeof clean, cudaMemcpyHostToDevice));
  DMB_CUDA_TRY(cudaMemcpy(ctx->aux, &clean, sizeof clean, cudaMemcpyHostToDevice));
  *out = ctx.release();
  return DMB_OK;
}

int dmb_ctx_destroy(dmb_ctx* ctx) {
  if (!ctx) return DMB_OK;
  cudaSetDevice(ctx->device);
  cudaFree(ctx->fb_list);
  cudaFree(ctx->fb_count);
  for (auto& kv : ctx->bases) {
    cudaFree(kv.second.tf32);
    cudaFree(kv.second.B);
    cudaFree(kv.second.BT);
    cudaFree(kv.second.B64);
  }
  RandomScratch& r = ctx->rnd;
  cudaFree(r.draws);
  cudaFree(r.first);
  cudaFree(r.second);
  cudaFree(r.bitmap);
  cudaFree(r.rank);
  cudaFree(r.idx);
  cudaFree(r.mt_seq);
  cudaFree(r.mt_windows);
  cudaFree(r.mt_reject);
  cudaFree(ctx->scratch);
  cudaFree(ctx->status);
  cudaFree(ctx->aux);
  delete ctx;
  return DMB_OK;
}

uint64_t dmb_wire_bytes(uint64_t n_values, uint64_t n_indices, int32_t dtype) {
  return wire_bytes(n_values, n_indices, dtype);
}
uint64_t dmb_period(double compression) { return period_of(compression); }

int dmb_plan_update(const dmb_rep_cfg* cfg, uint64_t len, uint64_t step, uint32_t shard,
                    dmb_update* out) {
  if (!cfg || !out) return fail(DMB_CONFIG, "NULL argument");
  return plan(cfg, len, step, shard, out);
}

uint64_t dmb_update_capacity(const dmb_rep_cfg* cfg, uint64_t len) { return capacity(cfg, len); }

int dmb_selected_indices(dmb_ctx* ctx, const dmb_rep_cfg* cfg, uint64_t step, uint32_t shard,
                         uint64_t len, uint32_t* d_out, uint64_t* count, void* stream) {
  cudaStream_t s = as_stream(stream);
  if (cfg->scheme != DMB_RANDOM && cfg->scheme != DMB_STRIDING)
    return fail(DMB_CONFIG, "selected_indices applies to random and striding schemes only");
  dmb_update u{};
  if (int rc = plan(cfg, len, step, shard, &u)) return rc;
  *count = u.n_values;
  if (cfg->scheme == DMB_RANDOM) {
    if (int rc = ensure_random(ctx, cfg, step, shard, len, u.n_values, s)) return rc;
    if (u.n_values)
      DMB_CUDA_TRY(cudaMemcpyAsync(d_out, ctx->rnd.idx, u.n_values * 4, cudaMemcpyDeviceToDevice, s));
    return DMB_OK;
  }
  // striding: o, o+n, ... < len (replicate.cpp:181-182)
  const uint64_t n = period_of(cfg->compression);
  launch_striding_iota(d_out, step % n, n, u.n_values, s);
  return last_launch();
}

int dmb_select_and_encode(dmb_ctx* ctx, const float* v, uint64_t len, const dmb_rep_cfg* cfg,
                          uint64_t step, uint32_t shard, dmb_update* out, float* local_q,
                          void* stream) {
  cudaStream_t s = as_stream(stream);
  if (int rc = clear_aux(ctx, s)) return rc;
  if (int rc = encode(ctx, ctx->aux, false, v, nullptr, nullptr, 0.0, len, cfg, step, shard, out,
                      local_q, nullptr, s))
    return rc;
  if (out->empty && local_q && len) DMB_CUDA_TRY(cudaMemsetAsync(local_q, 0, len * 4, s));
  return DMB_OK;
}

int dmb_decode_and_merge(dmb_ctx* ctx, const dmb_update* updates, uint64_t n_updates,
                         const dmb_rep_cfg* cfg, float* q, void* stream) {
  cudaStream_t s = as_stream(stream);
  if (int rc = validate_updates(updates, n_updates, cfg)) return rc;
  const dmb_update& r = updates[0];
  if (r.length == 0) return DMB_OK;
  if (int rc = clear_aux(ctx, s)) return rc;
  if (cfg->scheme == DMB_DEMO) {
    ChunkArgs a{};
    a.geo = geometry(cfg, r.length);
    if (int rc = get_basis(ctx, a.geo.s, &a.basis)) return rc;
    a.in = bodies_of(updates, n_updates, false);
    a.q_out = q;
    a.status = ctx->aux;
    launch_chunk_kernel(ChunkMode::MergeSgd, a, s);
    if (int rc = last_launch()) return rc;
    return check_aux_protocol(ctx, s);
  }
  SparseSel sel;
  if (int rc = sparse_sel(ctx, cfg, &r, &sel, s)) return rc;
  launch_sparse_merge_apply(sel, bodies_of(updates, n_updates, true), cfg->transfer_dtype,
                            kMergeOnly, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr,
                            nullptr, q, SgdScalars{}, AdamScalars{}, ctx->aux, s);
  return last_launch();
}

int dmb_serialize(const dmb_update* u, int32_t dtype, uint8_t* host_out, uint64_t cap,
                  uint64_t* written, void* stream) {
  // replicate.cpp:316-356: [tag u8][value count u64 LE][body]
  const uint64_t body = wire_bytes(u->n_values, u->scheme == DMB_DEMO ? u->n_indices : 0, dtype);
  if (cap < 9 + body) return fail(DMB_CONFIG, "serialize: buffer too small");
  host_out[0] = (uint8_t)u->scheme;
  for (int i = 0; i < 8; ++i) host_out[1 + i] = (uint8_t)(u->n_values >> (8 * i));
  if (body && is_mask(u)) {  // expand the exchange layout into the reference body
    std::vector<uint8_t> m(mask_body_bytes(u, dtype));
    DMB_CUDA_TRY(cudaMemcpyAsync(m.data(), u->body, m.size(), cudaMemcpyDeviceToHost, as_stream(stream)));
    DMB_CUDA_TRY(cudaStreamSynchronize(as_stream(stream)));
    const uint64_t nc = chunks_of(u), k = u->top_k;
    const uint8_t* vin = m.data() + 8 * nc;
    const int32_t vd = body_value_dtype(u, dtype);
    uint8_t* idx = host_out + 9;
    uint8_t* vout = idx + u->n_indices * 4;
    if (dtype == DMB_TERNARY) std::memset(vout, 0, (u->n_values * 2 + 7) / 8);
    for (uint64_t c = 0; c < nc; ++c) {
      uint64_t mk;
      std::memcpy(&mk, m.data() + 8 * c, 8);
      uint64_t t = c * k;
      for (uint32_t j = 0; j < 64 && mk; ++j, mk >>= 1) {
        if (!(mk & 1)) continue;
        std::memcpy(idx + 4 * t, &j, 4);
        float v;
        if (vd == DMB_TERNARY) {  // quad-order code words: 16 bytes per chunk
          uint32_t word;
          std::memcpy(&word, vin + 16 * c + 4 * ((j >> 1) & 3), 4);
          const uint32_t code = (word >> (2 * (2 * (j >> 3) + (j & 1)))) & 3u;
          v = code == 1u ? 1.0f : (code == 2u ? -1.0f : 0.0f);
        } else if (vd == DMB_FP16) {
          uint16_t h;
          std::memcpy(&h, vin + 2 * t, 2);
          v = half_to_float(h);
        } else {
          std::memcpy(&v, vin + 4 * t, 4);
        }
        if (dtype == DMB_FP32) std::memcpy(vout + 4 * t, &v, 4);
        else if (dtype == DMB_FP16) { const uint16_t h = float_to_half(v); std::memcpy(vout + 2 * t, &h, 2); }
        else { const uint32_t code = v > 0.0f ? 1u : (v < 0.0f ? 2u : 0u); vout[t >> 2] |= (uint8_t)(code << (2 * (t & 3))); }
        ++t;
      }
    }
    *written = 9 + body;
    return DMB_OK;
  }
  if (body) {
    DMB_CUDA_TRY(cudaMemcpyAsync(host_out + 9, u->body, body, cudaMemcpyDeviceToHost, as_stream(stream)));
    DMB_CUDA_TRY(cudaStreamSynchronize(as_stream(stream)));
  }
  *written = 9 + body;
  return DMB_OK;
}

int dmb_deserialize(const uint8_t* buf, uint64_t size, int32_t dtype, const dmb_update* tmpl,
                    dmb_update* out, void* stream) {
  // replicate.cpp:358-417, same checks and messages
  if (size < 9) return fail(DMB_PROTOCOL, "serialized update shorter than its header");
  const uint8_t tag = buf[0];
  if (tag < 1 || tag > 5) return fail(DMB_PROTOCOL, "unknown scheme tag");
  if ((int)tag != tmpl->scheme) return fail(DMB_PROTOCOL, "serialized scheme does not match the expected scheme");
  uint64_t count = 0;
  for (int i = 0; i < 8; ++i) count |= (uint64_t)buf[1 + i] << (8 * i);
  uint64_t off = 9;
  const uint64_t ni = tag == DMB_DEMO ? count : 0;
  if (tag == DMB_DEMO && size < off + count * 4) return fail(DMB_PROTOCOL, "truncated frequency indices");
  off += ni * 4;
  if (dtype == DMB_FP32 && size < off + count * 4) return fail(DMB_PROTOCOL, "truncated fp32 payload");
  if (dtype == DMB_FP16 && size < off + count * 2) return fail(DMB_PROTOCOL, "truncated fp16 payload");
  if (dtype == DMB_TERNARY && size < off + (count * 2 + 7) / 8) return fail(DMB_PROTOCOL, "truncated ternary payload");
  void* body = out->body;
  *out = *tmpl;
  out->body = body;
  out->n_values = count;
  out->n_indices = ni;
  out->empty = count == 0;
  out->bytes = wire_bytes(count, ni, dtype);
  if (out->bytes) {
    if (!body) return fail(DMB_CONFIG, "deserialize: output body is NULL");
    DMB_CUDA_TRY(cudaMemcpyAsync(body, buf + 9, out->bytes, cudaMemcpyHostToDevice, as_stream(stream)));
    DMB_CUDA_TRY(cudaStreamSynchronize(as_stream(stream)));
  }
  return DMB_OK;
}

int dmb_update_values(const dmb_update* u, int32_t dtype, float* d_values, void* stream) {
  if (u->n_values == 0) return DMB_OK;
  if (is_mask(u)) {  // inspection of an exchange-layout body: through the reference bytes
    std::vector<uint8_t> hb(9 + wire_bytes(u->n_values, u->n_indices, dtype));
    uint64_t written = 0;
    if (int rc = dmb_serialize(u, dtype, hb.data(), hb.size(), &written, stream)) return rc;
    std::vector<float> v(u->n_values);
    const uint8_t* vin = hb.data() + 9 + u->n_indices * 4;
    for (uint64_t t = 0; t < u->n_values; ++t) {
      if (dtype == DMB_FP32) std::memcpy(&v[t], vin + 4 * t, 4);
      else if (dtype == DMB_FP16) { uint16_t h; std::memcpy(&h, vin + 2 * t, 2); v[t] = half_to_float(h); }
      else { const uint32_t code = (vin[t >> 2] >> (2 * (t & 3))) & 3u; v[t] = code == 1u ? 1.0f : (code == 2u ? -1.0f : 0.0f); }
    }
    DMB_CUDA_TRY(cudaMemcpyAsync(d_values, v.data(), v.size() * 4, cudaMemcpyHostToDevice, as_stream(stream)));
    DMB_CUDA_TRY(cudaStreamSynchronize(as_stream(stream)));
    return DMB_OK;
  }
  launch_unpack_values(values_region(u), u->n_values, body_value_dtype(u, dtype), d_values, as_stream(stream));
  return last_launch();
}

int dmb_demo_sgd_prepare(dmb_ctx* ctx, const float* grad, const float* m_in, float* m_out,
                         uint64_t len, const dmb_opt_cfg* opt, const dmb_rep_cfg* cfg,
                         uint64_t step, uint32_t shard, dmb_update* out, float* local_q,
                         float* m_accum, void* stream) {
  cudaStream_t s = as_stream(stream);
  if (int rc = encode(ctx, ctx->status, true, grad, m_in, m_out, opt->momentum_decay, len, cfg,
                      step, shard, out, local_q, m_accum, s))
    return rc;
  if (out->empty && local_q && len) DMB_CUDA_TRY(cudaMemsetAsync(local_q, 0, len * 4, s));
  return DMB_OK;
}

int dmb_demo_sgd_prepare_members(dmb_ctx* ctx, const float* const* members, uint32_t n_members, float* grad_mean,
                                 const float* m_in, float* m_out, uint64_t len, const dmb_opt_cfg* opt,
                                 const dmb_rep_cfg* cfg, uint64_t step, uint32_t shard, dmb_update* out,
                                 void* stream) {
  cudaStream_t s = as_stream(stream);
  if (!members || n_members == 0 || n_members > (uint32_t)kMaxReplicas)
    return fail(DMB_PROTOCOL, "reduce-scatter over %u members", n_members);
  // the SGD modes take the mean as a pass of its own (their fused load is compiled out: it cost
  // the one-rank SGD step and measured slower in the cluster), then the prepare
  if (len) launch_grad_mean(members, (int)n_members, len, grad_mean, s);
  return dmb_demo_sgd_prepare(ctx, grad_mean, m_in, m_out, len, opt, cfg, step, shard, out, nullptr, nullptr,
                              stream);
}

int dmb_demo_sgd_apply(dmb_ctx* ctx, float* params, const float* q, uint64_t n, double lr,
                       void* stream) {
  if (!n) return DMB_OK;
  launch_sgd_apply(params, q, n, (float)lr, ctx->status, as_stream(stream));
  return last_launch();
}

int dmb_adamw_prepare(dmb_ctx* ctx, const float* grad, uint64_t len, const dmb_rep_cfg* cfg,
                      uint64_t step, uint32_t shard, dmb_update* out, float* local_q,
                      void* stream) {
  cudaStream_t s = as_stream(stream);
  if (int rc = encode(ctx, ctx->status, false, grad, nullptr, nullptr, 0.0, len, cfg, step, shard,
                      out, local_q, nullptr, s))
    return rc;
  if (out->empty) {
    // no kernel ran over grad: still enforce require_finite (optim.cpp:53)
    if (len) launch_check_finite(grad, len, ctx->status, s);
    if (local_q && len) DMB_CUDA_TRY(cudaMemsetAsync(local_q, 0, len * 4, s));
    return last_launch();
  }
  return DMB_OK;
}

int dmb_adamw_prepare_members(dmb_ctx* ctx, const float* const* members, uint32_t n_members, float* grad_mean,
                              uint64_t len, const dmb_rep_cfg* cfg, uint64_t step, uint32_t shard,
                              dmb_update* out, void* stream) {
  cudaStream_t s = as_stream(stream);
  if (!members || n_members == 0 || n_members > (uint32_t)kMaxReplicas)
    return fail(DMB_PROTOCOL, "reduce-scatter over %u members", n_members);
  if (cfg->scheme != DMB_DEMO || n_members > (uint32_t)kMaxGradSrc) {  // the mean first, then the prepare
    if (len) launch_grad_mean(members, (int)n_members, len, grad_mean, s);
    return dmb_adamw_prepare(ctx, grad_mean, len, cfg, step, shard, out, nullptr, stream);
  }
  return encode(ctx, ctx->status, false, grad_mean, nullptr, nullptr, 0.0, len, cfg, step, shard, out, nullptr,
                nullptr, s, members, (int)n_members);
}

int dmb_adamw_apply(dmb_ctx* ctx, float* params, float* exp_avg, float* exp_avg_sq,
                    uint64_t* steps, const float* grad, const float* local_q, const float* merged,
                    uint64_t n, const dmb_opt_cfg* opt, double lr, void* stream) {
  *steps += 1;
  if (!n) return DMB_OK;
  launch_adamw_apply(params, exp_avg, exp_avg_sq, grad, local_q, merged, n,
                     adam_scalars(opt, *steps, lr), ctx->status, as_stream(stream));
  return last_launch();
}

int dmb_baseline_sgd_step(dmb_ctx* ctx, float* params, float* m, const float* grad, uint64_t n,
                          const dmb_opt_cfg* opt, double lr, void* stream) {
  if (!n) return DMB_OK;
  launch_baseline_sgd(params, m, grad, n, (float)opt->momentum_decay, (float)lr, ctx->status,
                      as_stream(stream));
  return last_launch();
}

namespace {
int merge_sgd(dmb_ctx* ctx, const dmb_update* updates, uint64_t n_updates, const dmb_rep_cfg* cfg,
              const float* p_in, float* params, uint64_t len, double lr, cudaStream_t s);
int merge_adamw(dmb_ctx* ctx, const dmb_update* updates, uint64_t n_updates, uint64_t own_rank,
                const dmb_rep_cfg* cfg, const float* p_in, float* p_out, const float* ea_in, float* ea_out,
                const float* es_in, float* es_out, uint64_t* steps, const float* grad, uint64_t len,
                const dmb_opt_cfg* opt, double lr, cudaStream_t s);
}  // namespace

int dmb_merge_apply_sgd(dmb_ctx* ctx, const dmb_update* updates, uint64_t n_updates,
                        const dmb_rep_cfg* cfg, float* params, const float* grad_if_unsynced,
                        uint64_t len, uint64_t step, double lr, void* stream) {
  (void)step;
  if (!updates || n_updates == 0 || updates[0].empty) {
    // DiLoCo between beats: SGD steps on the raw shard gradient (cluster.cpp:225)
    if (!grad_if_unsynced) return fail(DMB_PROTOCOL, "unsynced step needs the local gradient");
    return dmb_demo_sgd_apply(ctx, params, grad_if_unsynced, len, lr, stream);
  }
  return merge_sgd(ctx, updates, n_updates, cfg, params, params, len, lr, as_stream(stream));
}

int dmb_merge_apply_sgd_to(dmb_ctx* ctx, const dmb_update* updates, uint64_t n_updates,
                           const dmb_rep_cfg* cfg, const float* p_in, float* p_out, uint64_t len,
                           uint64_t step, double lr, void* stream) {
  (void)step;
  if (!updates || n_updates == 0 || updates[0].empty)
    return fail(DMB_PROTOCOL, "the out-of-place merge needs synchronized updates");
  return merge_sgd(ctx, updates, n_updates, cfg, p_in, p_out, len, lr, as_stream(stream));
}

int dmb_merge_apply_adamw_to(dmb_ctx* ctx, const dmb_update* updates, uint64_t n_updates,
                             uint64_t own_rank, const dmb_rep_cfg* cfg, const float* p_in, float* p_out,
                             const float* ea_in, float* ea_out, const float* es_in, float* es_out,
                             uint64_t* steps, const float* grad, uint64_t len, uint64_t step,
                             const dmb_opt_cfg* opt, double lr, void* stream) {
  (void)step;
  if (!updates || n_updates == 0 || updates[0].empty)
    return fail(DMB_PROTOCOL, "the out-of-place merge needs synchronized updates");
  return merge_adamw(ctx, updates, n_updates, own_rank, cfg, p_in, p_out, ea_in, ea_out, es_in, es_out, steps,
                     grad, len, opt, lr, as_stream(stream));
}

namespace {
int merge_sgd(dmb_ctx* ctx, const dmb_update* updates, uint64_t n_updates, const dmb_rep_cfg* cfg,
              const float* p_in, float* params, uint64_t len, double lr, cudaStream_t s) {
  if (int rc = validate_updates(updates, n_updates, cfg)) return rc;
  if (updates[0].length != len) return fail(DMB_PROTOCOL, "update length does not match the shard");
  if (!len) return DMB_OK;
  if (cfg->scheme == DMB_DEMO) {
    ChunkArgs a{};
    a.geo = geometry(cfg, len);
    if (int rc = get_basis(ctx, a.geo.s, &a.basis)) return rc;
    a.in = bodies_of(updates, n_updates, false);
    a.p_in = p_in;
    a.p_out = params;
    a.sgd = sgd_scalars(0.0, lr);
    a.status = ctx->status;
    if (int rc = attach_fallback(ctx, &a)) return rc;
    if (is_mask(&updates[0])) {
      if (!(len % cfg->chunk_size == 0 && tc_enabled() && tc3_supported(ChunkMode::MergeSgd, a)))
        return fail(DMB_PROTOCOL, "mask-format updates need the tensor-core merge path (s = 64, whole chunks)");
      a.geo.wire_mask = 1;
    }
    launch_chunk_kernel(ChunkMode::MergeSgd, a, s);
    return last_launch();
  }
  SparseSel sel;
  if (int rc = sparse_sel(ctx, cfg, &updates[0], &sel, s)) return rc;
  launch_sparse_merge_apply(sel, bodies_of(updates, n_updates, true), cfg->transfer_dtype,
                            kMergeSgd, nullptr, p_in, params, nullptr, nullptr, nullptr, nullptr,
                            nullptr, sgd_scalars(0.0, lr), AdamScalars{}, ctx->status, s);
  return last_launch();
}
}  // namespace

int dmb_merge_apply_adamw(dmb_ctx* ctx, const dmb_update* updates, uint64_t n_updates,
                          uint64_t own_rank, const dmb_rep_cfg* cfg, float* params,
                          float* exp_avg, float* exp_avg_sq, uint64_t* steps, const float* grad,
                          uint64_t len, uint64_t step, const dmb_opt_cfg* opt, double lr,
                          void* stream) {
  (void)step;
  if (!updates || n_updates == 0 || updates[0].empty) {
    // merged == nullptr: AdamW on the raw local gradient (cluster.cpp:227, optim.cpp:65)
    return dmb_adamw_apply(ctx, params, exp_avg, exp_avg_sq, steps, grad, grad, nullptr, len, opt,
                           lr, stream);
  }
  return merge_adamw(ctx, updates, n_updates, own_rank, cfg, params, params, exp_avg, exp_avg, exp_avg_sq,
                     exp_avg_sq, steps, grad, len, opt, lr, as_stream(stream));
}

namespace {
int merge_adamw(dmb_ctx* ctx, const dmb_update* updates, uint64_t n_updates, uint64_t own_rank,
                const dmb_rep_cfg* cfg, const float* p_in, float* params, const float* ea_in, float* exp_avg,
                const float* es_in, float* exp_avg_sq, uint64_t* steps, const float* grad, uint64_t len,
                const dmb_opt_cfg* opt, double lr, cudaStream_t s) {
  if (int rc = validate_updates(updates, n_updates, cfg)) return rc;
  if (updates[0].length != len) return fail(DMB_PROTOCOL, "update length does not match the shard");
  if (own_rank >= n_updates) return fail(DMB_PROTOCOL, "own rank outside the replica group");
  *steps += 1;
  if (!len) return DMB_OK;
  const AdamScalars A = adam_scalars(opt, *steps, lr);
  if (cfg->scheme == DMB_DEMO) {
    ChunkArgs a{};
    a.geo = geometry(cfg, len);
    if (int rc = get_basis(ctx, a.geo.s, &a.basis)) return rc;
    a.in = bodies_of(updates, n_updates, false);
    a.own_rank = (int)own_rank;
    a.g = grad;
    a.p_in = p_in;
    a.p_out = params;
    a.ea_in = ea_in;
    a.ea_out = exp_avg;
    a.es_in = es_in;
    a.es_out = exp_avg_sq;
    a.adam = A;
    a.status = ctx->status;
    if (int rc = attach_fallback(ctx, &a)) return rc;
    if (is_mask(&updates[0])) {
      if (!(len % cfg->chunk_size == 0 && tc_enabled() && tc3_supported(ChunkMode::MergeAdam, a)))
        return fail(DMB_PROTOCOL, "mask-format updates need the tensor-core merge path (s = 64, whole chunks)");
      a.geo.wire_mask = 1;
    }
    launch_chunk_kernel(ChunkMode::MergeAdam, a, s);
    return last_launch();
  }
  SparseSel sel;
  if (int rc = sparse_sel(ctx, cfg, &updates[0], &sel, s)) return rc;
  launch_sparse_merge_apply(sel, bodies_of(updates, n_updates, true), cfg->transfer_dtype,
                            kMergeAdam, grad, p_in, params, ea_in, exp_avg, es_in,
                            exp_avg_sq, nullptr, SgdScalars{}, A, ctx->status, s);
  return last_launch();
}
}  // namespace

int dmb_step_sgd_local(dmb_ctx* ctx, const float* grad, const float* m_in, float* m_out,
                       const float* p_in, float* p_out, uint64_t len, const dmb_opt_cfg* opt,
                       const dmb_rep_cfg* cfg, uint64_t step, uint32_t shard, double lr,
                       dmb_update* out, void* stream) {
  cudaStream_t s = as_stream(stream);
  dmb_update hdr{};
  if (out) hdr.body = out->body;
  if (int rc = plan(cfg, len, step, shard, &hdr)) return rc;
  if (out) *out = hdr;
  if (!len) return DMB_OK;
  if (cfg->scheme == DMB_DEMO) {
    if (out && out->body) {
      if (int rc = prep_values_region(out, cfg->transfer_dtype, s)) return rc;
    }
    ChunkArgs a{};
    a.geo = geometry(cfg, len);
    if (int rc = get_basis(ctx, a.geo.s, &a.basis)) return rc;
    a.g = grad;
    a.m_in = m_in;
    a.m_out = m_out;
    a.p_in = p_in;
    a.p_out = p_out;
    a.body = out ? static_cast<uint8_t*>(out->body) : nullptr;
    a.sgd = sgd_scalars(opt->momentum_decay, lr);
    a.status = ctx->status;
    if (int rc = attach_fallback(ctx, &a)) return rc;
    launch_chunk_kernel(ChunkMode::StepSgd, a, s);
    return last_launch();
  }
  return fail(DMB_CONFIG, "the fused one-member step covers the demo scheme; use prepare + merge_apply");
}

int dmb_step_sgd_local_members(dmb_ctx* ctx, const float* const* members, uint32_t n_members, float* grad_mean,
                               const float* m_in, float* m_out, const float* p_in, float* p_out, uint64_t len,
                               const dmb_opt_cfg* opt, const dmb_rep_cfg* cfg, uint64_t step, uint32_t shard,
                               double lr, dmb_update* out, void* stream) {
  cudaStream_t s = as_stream(stream);
  if (!members || n_members == 0 || n_members > (uint32_t)kMaxReplicas)
    return fail(DMB_PROTOCOL, "reduce-scatter over %u members", n_members);
  if (len) launch_grad_mean(members, (int)n_members, len, grad_mean, s);  // a pass of its own (SGD)
  return dmb_step_sgd_local(ctx, grad_mean, m_in, m_out, p_in, p_out, len, opt, cfg, step, shard, lr, out, stream);
}

int dmb_step_adamw_local(dmb_ctx* ctx, const float* grad, const float* p_in, float* p_out,
                         const float* ea_in, float* ea_out, const float* es_in, float* es_out,
                         uint64_t* steps, uint64_t len, const dmb_opt_cfg* opt,
                         const dmb_rep_cfg* cfg, uint64_t step, uint32_t shard, double lr,
                         dmb_update* out, void* stream) {
  cudaStream_t s = as_stream(stream);
  dmb_update hdr{};
  if (out) hdr.body = out->body;
  if (int rc = plan(cfg, len, step, shard, &hdr)) return rc;
  if (out) *out = hdr;
  if (cfg->scheme != DMB_DEMO)
    return fail(DMB_CONFIG, "the fused one-member step covers the demo scheme; use prepare + merge_apply");
  *steps += 1;
  if (!len) return DMB_OK;
  if (out && out->body) {
    if (int rc = prep_values_region(out, cfg->transfer_dtype, s)) return rc;
  }
  ChunkArgs a{};
  a.geo = geometry(cfg, len);
  if (int rc = get_basis(ctx, a.geo.s, &a.basis)) return rc;
  a.g = grad;
  a.p_in = p_in;
  a.p_out = p_out;
  a.ea_in = ea_in;
  a.ea_out = ea_out;
  a.es_in = es_in;
  a.es_out = es_out;
  a.body = out ? static_cast<uint8_t*>(out->body) : nullptr;
  a.adam = adam_scalars(opt, *steps, lr);
  a.status = ctx->status;
  if (int rc = attach_fallback(ctx, &a)) return rc;
  launch_chunk_kernel(ChunkMode::StepAdam, a, s);
  return last_launch();
}

int dmb_step_adamw_local_members(dmb_ctx* ctx, const float* const* members, uint32_t n_members, float* grad_mean,
                                 const float* p_in, float* p_out, const float* ea_in, float* ea_out,
                                 const float* es_in, float* es_out, uint64_t* steps, uint64_t len,
                                 const dmb_opt_cfg* opt, const dmb_rep_cfg* cfg, uint64_t step, uint32_t shard,
                                 double lr, dmb_update* out, void* stream) {
  cudaStream_t s = as_stream(stream);
  if (!members || n_members == 0 || n_members > (uint32_t)kMaxReplicas)
    return fail(DMB_PROTOCOL, "reduce-scatter over %u members", n_members);
  if (n_members > 2) {  // the fused load takes two members next to the state staging
    if (len) launch_grad_mean(members, (int)n_members, len, grad_mean, s);
    return dmb_step_adamw_local(ctx, grad_mean, p_in, p_out, ea_in, ea_out, es_in, es_out, steps, len, opt, cfg,
                                step, shard, lr, out, stream);
  }
  dmb_update hdr{};
  if (out) hdr.body = out->body;
  if (int rc = plan(cfg, len, step, shard, &hdr)) return rc;
  if (out) *out = hdr;
  if (cfg->scheme != DMB_DEMO)
    return fail(DMB_CONFIG, "the fused one-member step covers the demo scheme; use prepare + merge_apply");
  *steps += 1;
  if (!len) return DMB_OK;
  if (out && out->body) {
    if (int rc = prep_values_region(out, cfg->transfer_dtype, s)) return rc;
  }
  ChunkArgs a{};
  a.geo = geometry(cfg, len);
  if (int rc = get_basis(ctx, a.geo.s, &a.basis)) return rc;
  a.g = grad_mean;
  a.n_src = (int)n_members;
  for (uint32_t q = 0; q < n_members; ++q) a.g_src[q] = members[q];
  a.p_in = p_in;
  a.p_out = p_out;
  a.ea_in = ea_in;
  a.ea_out = ea_out;
  a.es_in = es_in;
  a.es_out = es_out;
  a.body = out ? static_cast<uint8_t*>(out->body) : nullptr;
  a.adam = adam_scalars(opt, *steps, lr);
  a.status = ctx->status;
  if (int rc = attach_fallback(ctx, &a)) return rc;
  launch_chunk_kernel(ChunkMode::StepAdam, a, s);
  return last_launch();
}

int dmb_grad_mean(dmb_ctx* ctx, const float* const* grads, uint64_t members, uint64_t len,
                  float* out, void* stream) {
  (void)ctx;
  if (members == 0) return fail(DMB_PROTOCOL, "reduce-scatter over an empty group");
  if (members > (uint64_t)kMaxReplicas) return fail(DMB_PROTOCOL, "too many members");
  if (!len) return DMB_OK;
  launch_grad_mean(grads, (int)members, len, out, as_stream(stream));
  return last_launch();
}

int dmb_grad_mean_pull(dmb_ctx* ctx, const float* const* grads, uint64_t members, uint64_t len, float* out,
                       uint32_t ctas, void* stream) {
  (void)ctx;
  if (members == 0) return fail(DMB_PROTOCOL, "reduce-scatter over an empty group");
  if (members > (uint64_t)kMaxReplicas) return fail(DMB_PROTOCOL, "too many members");
  if (!len) return DMB_OK;
  launch_grad_mean_pull(grads, (int)members, len, out, (int)ctas, as_stream(stream));
  return last_launch();
}

int dmb_require_finite(dmb_ctx* ctx, const float* v, uint64_t n, void* stream) {
  if (!n) return DMB_OK;
  launch_check_finite(v, n, ctx->status, as_stream(stream));
  return last_launch();
}

int dmb_status(dmb_ctx* ctx, void* stream, int64_t* first_bad) {
  cudaStream_t s = as_stream(stream);
  DevStatus h{};
  DMB_CUDA_TRY(cudaMemcpyAsync(&h, ctx->status, sizeof h, cudaMemcpyDeviceToHost, s));
  DMB_CUDA_TRY(cudaStreamSynchronize(s));
  if (first_bad) *first_bad = h.first_bad == kNoBad ? -1 : (int64_t)h.first_bad;
  if (h.protocol_error) {
    DMB_CUDA_TRY(cudaMemset(&ctx->status->protocol_error, 0, sizeof(unsigned int)));
    return fail(DMB_PROTOCOL, "frequency index out of range");
  }
  if (h.first_bad == kPeerBad) {
    DMB_CUDA_TRY(cudaMemset(&ctx->status->first_bad, 0xff, sizeof(unsigned long long)));
    if (first_bad) *first_bad = -2;
    return fail(DMB_TRAINING, "gradient contains a non-finite value (on another rank of the step)");
  }
  if (h.first_bad != kNoBad) {
    DMB_CUDA_TRY(cudaMemset(&ctx->status->first_bad, 0xff, sizeof(unsigned long long)));
    return fail(DMB_TRAINING, "gradient contains a non-finite value (at index %llu)",
                (unsigned long long)h.first_bad);
  }
  return DMB_OK;
}

int dmb_fallback_chunks(dmb_ctx* ctx, void* stream, uint64_t* count) {
  DevStatus a{}, b{};
  DMB_CUDA_TRY(cudaMemcpyAsync(&a, ctx->status, sizeof a, cudaMemcpyDeviceToHost, as_stream(stream)));
  DMB_CUDA_TRY(cudaMemcpyAsync(&b, ctx->aux, sizeof b, cudaMemcpyDeviceToHost, as_stream(stream)));
  DMB_CUDA_TRY(cudaStreamSynchronize(as_stream(stream)));
  *count = a.fallback_chunks + b.fallback_chunks;
  return DMB_OK;
}

// ---- transform.hpp:13-74 -------------------------------------------------------
int dmb_chunk_layout(uint64_t length, uint64_t chunk_size, dmb_layout* out) {
  if (!out) return fail(DMB_CONFIG, "NULL argument");
  if (chunk_size == 0) return fail(DMB_CONFIG, "chunk size must be positive");  // transform.cpp:18
  out->length = length;
  out->chunk_size = chunk_size;
  out->num_chunks = (length + chunk_size - 1) / chunk_size;
  out->pad = out->num_chunks * chunk_size - length;
  return DMB_OK;
}

int dmb_chunk(dmb_ctx* ctx, const float* v, const dmb_layout* layout, float* rows, void* stream) {
  (void)ctx;
  if (!layout || layout->chunk_size == 0) return fail(DMB_CONFIG, "chunk: layout does not match the vector");
  const uint64_t padded = layout->num_chunks * layout->chunk_size;
  if (padded) launch_chunk(v, layout->length, padded, rows, as_stream(stream));
  return last_launch();
}

int dmb_unchunk(dmb_ctx* ctx, const float* rows, const dmb_layout* layout, float* v, void* stream) {
  (void)ctx;
  if (!layout || layout->chunk_size == 0) return fail(DMB_CONFIG, "unchunk: row buffer does not match the layout");
  if (layout->length) launch_copy(rows, layout->length, v, as_stream(stream));
  return last_launch();
}

static int dct_common(dmb_ctx* ctx, bool inverse, const float* in, uint64_t size, uint64_t count, float* out,
                      void* stream) {
  if (size == 0) return fail(DMB_CONFIG, "transform size must be positive");  // transform.cpp:43
  if (size > 1024) return fail(DMB_CONFIG, "transform size %llu above the device limit 1024", (unsigned long long)size);
  if (!count) return DMB_OK;
  Basis b{};
  if (int rc = get_basis(ctx, (int)size, &b)) return rc;
  launch_dct(inverse, in, size, count, b, out, as_stream(stream));
  return last_launch();
}

int dmb_dct2(dmb_ctx* ctx, const float* x, uint64_t size, uint64_t count, float* out, void* stream) {
  return dct_common(ctx, false, x, size, count, out, stream);
}

int dmb_idct3(dmb_ctx* ctx, const float* coeffs, uint64_t size, uint64_t count, float* out, void* stream) {
  return dct_common(ctx, true, coeffs, size, count, out, stream);
}

int dmb_sign_transform(dmb_ctx* ctx, float* v, uint64_t n, void* stream) {
  (void)ctx;
  if (n) launch_sign(v, n, as_stream(stream));
  return last_launch();
}

// ---- model.hpp toy producers (toy_models.cu) ---------------------------------------
namespace {
int toy_args(const dmb_toy_model* m, const dmb_toy_pool* pool, ToyArgs& a) {
  if (!m || !pool) return fail(DMB_CONFIG, "model and pool are required");
  if (m->kind > 1) return fail(DMB_CONFIG, "unknown model kind %u", m->kind);
  if (m->n_dims == 0 || m->n_dims > (uint32_t)kToyMaxDims || (m->kind == 0 && m->n_dims != 1) ||
      (m->kind == 1 && m->n_dims < 2))
    return fail(DMB_CONFIG, "model dims: a quadratic model takes one, an mlp 2..%d", kToyMaxDims);
  for (uint32_t l = 0; l < m->n_dims; ++l)
    if (m->dims[l] == 0) return fail(DMB_CONFIG, "model dims must be positive");
  if (m->kind == 1 && m->loss == 1 && !pool->labels)
    return fail(DMB_CONFIG, "cross entropy batch is missing labels");  // model.cpp:24-27
  if (m->kind == 1 && m->loss == 0 && !pool->targets)
    return fail(DMB_CONFIG, "regression batch targets do not match model output dim");  // model.cpp:28-30
  if (!pool->inputs || pool->size == 0) return fail(DMB_CONFIG, "empty batch");  // model.cpp:20
  a = ToyArgs{};
  a.kind = (int)m->kind;
  a.activation = (int)m->activation;
  a.loss_kind = (int)m->loss;
  a.n_dims = m->n_dims;
  for (uint32_t l = 0; l < m->n_dims; ++l) a.dims[l] = m->dims[l];
  a.inputs = pool->inputs;
  a.targets = pool->targets;
  a.labels = pool->labels;
  return DMB_OK;
}
uint64_t toy_param_count(const dmb_toy_model* m) {  // model.cpp:121-125
  if (m->kind == 0) return m->dims[0];
  uint64_t n = 0;
  for (uint32_t l = 0; l + 1 < m->n_dims; ++l) n += (uint64_t)m->dims[l + 1] * m->dims[l] + m->dims[l + 1];
  return n;
}
int toy_launch(const ToyArgs& a, cudaStream_t s) {
  if (toy_smem_bytes(a) > 227 * 1024)
    return fail(DMB_CONFIG, "toy producer: %llu B of shared memory (gradient + activations) exceed the 227 KB of an SM",
                (unsigned long long)toy_smem_bytes(a));
  launch_toy(a, s);
  return last_launch();
}
}  // namespace

int dmb_toy_loss_grad(dmb_ctx* ctx, const dmb_toy_model* model, const dmb_toy_pool* pool, const int64_t* order,
                      uint64_t step, uint64_t batch, const float* params, uint64_t params_stride,
                      uint64_t workers_per_row, uint64_t workers, float* grad, uint64_t grad_len, double* loss,
                      void* stream) {
  (void)ctx;
  ToyArgs a;
  if (int rc = toy_args(model, pool, a)) return rc;
  if (batch == 0) return fail(DMB_CONFIG, "empty batch");
  if (workers == 0 || workers_per_row == 0) return fail(DMB_CONFIG, "no workers");
  if (workers * batch > pool->size)  // dataset.cpp:127-133
    return fail(DMB_CONFIG, "global batch %llu x %llu exceeds the training pool of %llu examples",
                (unsigned long long)workers, (unsigned long long)batch, (unsigned long long)pool->size);
  if (grad_len < toy_param_count(model) || params_stride < toy_param_count(model))
    return fail(DMB_CONFIG, "parameter vector too short: %llu < %llu", (unsigned long long)params_stride,
                (unsigned long long)toy_param_count(model));  // model.cpp:15-19
  if (!order) return fail(DMB_CONFIG, "the batch permutation is required");
  a.order = order;
  a.order_len = pool->size;
  a.step = step;
  a.world = workers;
  a.batch = batch;
  a.params = params;
  a.params_stride = params_stride;
  a.workers_per_row = workers_per_row;
  a.workers = workers;
  a.grad = grad;
  a.grad_stride = grad_len;
  a.grad_len = grad_len;
  a.loss = loss;
  return toy_launch(a, as_stream(stream));
}

int dmb_toy_loss(dmb_ctx* ctx, const dmb_toy_model* model, const dmb_toy_pool* pool, const float* params,
                 double* loss, void* stream) {
  (void)ctx;
  ToyArgs a;
  if (int rc = toy_args(model, pool, a)) return rc;
  a.order = nullptr;
  a.batch = pool->size;
  a.world = 1;
  a.params = params;
  a.params_stride = toy_param_count(model);
  a.workers_per_row = 1;
  a.workers = 1;
  a.loss = loss;
  return toy_launch(a, as_stream(stream));
}

int dmb_extract_fast_components(dmb_ctx* ctx, const float* v, uint64_t len, uint64_t chunk_size, uint64_t top_k,
                                uint32_t* indices, float* coeffs, float* fast, float* residual, void* stream) {
  cudaStream_t s = as_stream(stream);
  if (top_k == 0 || top_k > chunk_size)  // transform.cpp:96-101
    return fail(DMB_CONFIG, "top_k %llu out of range for chunk size %llu", (unsigned long long)top_k,
                (unsigned long long)chunk_size);
  dmb_rep_cfg cfg{};
  cfg.scheme = DMB_DEMO;
  cfg.sign_mode = 0;
  cfg.transfer_dtype = DMB_FP32;  // fp32 values are the coefficients, not narrowed (replicate.cpp:137-144)
  cfg.chunk_size = chunk_size;
  cfg.top_k = top_k;
  cfg.compression = (double)top_k / (double)chunk_size;
  const uint64_t cap = capacity(&cfg, len);
  if (cap > ctx->scratch_cap) {
    cudaFree(ctx->scratch);
    DMB_CUDA_TRY(cudaMalloc(&ctx->scratch, cap));
    ctx->scratch_cap = cap;
  }
  dmb_update u{};
  u.body = ctx->scratch;
  const int wf = ctx->wire_format;
  ctx->wire_format = DMB_WIRE_REFERENCE;
  if (int rc = clear_aux(ctx, s)) return rc;
  const int rc = encode(ctx, ctx->aux, false, v, nullptr, nullptr, 0.0, len, &cfg, 0, 0, &u, fast, nullptr, s);
  ctx->wire_format = wf;
  if (rc) return rc;
  const uint64_t n = u.n_values;  // num_chunks * top_k
  if (n) {
    if (indices) DMB_CUDA_TRY(cudaMemcpyAsync(indices, ctx->scratch, n * 4, cudaMemcpyDeviceToDevice, s));
    if (coeffs) DMB_CUDA_TRY(cudaMemcpyAsync(coeffs, ctx->scratch + n * 4, n * 4, cudaMemcpyDeviceToDevice, s));
  }
  if (residual && len) launch_residual(v, fast, len, top_k == chunk_size, residual, s);
  return last_launch();
}

// test hook (not in the public header): the MT19937-64 jump-ahead of substream b, on the host
int dmb_debug_mt_jump_check(uint64_t engine_seed, uint64_t b) {
  const char* err = nullptr;
  const int rc = mt_jump_check(engine_seed, b, &err);
  if (rc < 0) return fail(DMB_CUDA, "%s", err ? err : "jump table");
  return rc;
}

// tuning hook (not in the public header): device buffer of 32 x 16 u64 timestamps
void dmb_debug_events(unsigned long long* d_buf) { g_dbg = d_buf; }

int dmb_set_sm_reserve(int sms) {
  if (sms < 0) return fail(DMB_CONFIG, "negative SM reserve");
  g_sm_reserve.store(sms, std::memory_order_relaxed);
  return DMB_OK;
}

int dmb_kernel_timer_enable(int on) {
  std::lock_guard<std::mutex> l(g_timer_mu);
  g_timer_on = on != 0;
  return DMB_OK;
}

int dmb_kernel_timer_read(double* total_ms, uint64_t* launches) {
  std::lock_guard<std::mutex> l(g_timer_mu);
  double t = 0.0;
  uint64_t n = 0;
  for (auto& pr : g_timer_pairs) {
    float ms = 0.f;
    if (cudaEventSynchronize(pr.second) == cudaSuccess && cudaEventElapsedTime(&ms, pr.first, pr.second) == cudaSuccess) {
      t += ms;
      ++n;
    }
    g_timer_pool.push_back(pr);
  }
  g_timer_pairs.clear();
  if (total_ms) *total_ms = t;
  if (launches) *launches = n;
  return DMB_OK;
}

int dmb_plan_exchange(dmb_ctx* ctx, const dmb_rep_cfg* cfg, uint64_t len, uint64_t step, uint32_t shard,
                      dmb_update* out) {
  if (!ctx || !cfg || !out) return fail(DMB_CONFIG, "NULL argument");
  if (int rc = plan(cfg, len, step, shard, out)) return rc;
  if (!out->empty && mask_layout(ctx, cfg, len)) set_mask_header(cfg, out);
  return DMB_OK;
}

int dmb_latch_export(dmb_ctx* ctx, int32_t* d_flag, void* stream) {
  if (!ctx || !d_flag) return fail(DMB_CONFIG, "NULL argument");
  latch_export_kernel<<<1, 1, 0, as_stream(stream)>>>(ctx->status, d_flag);
  count_launches(1);
  return last_launch();
}

int dmb_latch_import(dmb_ctx* ctx, const int32_t* d_flag, void* stream) {
  if (!ctx || !d_flag) return fail(DMB_CONFIG, "NULL argument");
  latch_import_kernel<<<1, 1, 0, as_stream(stream)>>>(ctx->status, d_flag);
  count_launches(1);
  return last_launch();
}

int dmb_set_wire_format(dmb_ctx* ctx, int32_t format) {
  if (!ctx) return fail(DMB_CONFIG, "ctx is NULL");
  if (format != DMB_WIRE_REFERENCE && format != DMB_WIRE_MASK) return fail(DMB_CONFIG, "unknown wire format %d", format);
  ctx->wire_format = format;
  return DMB_OK;
}

uint64_t dmb_launch_count(dmb_ctx* ctx) {
  (void)ctx;
  return g_launches.load();
}

}  // extern "C"
