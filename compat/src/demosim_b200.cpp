// demosim_b200.cpp -- the reference's C++ API (namespace demosim: transform.hpp, replicate.hpp,
// optim.hpp, vec.hpp, rng.hpp; the quadratic toy model of model.hpp) implemented over the
// B200 C ABI (include/demo_b200.h), so code written against /root/reference/proj/core links
// against the device path unchanged.  Host FP64 vectors cross to the device as FP32
// (to_device / from_device); errors come back as the reference's exception classes
// (common.hpp:10-26) with the library's message.  One context on device 0, the legacy
// default stream, synchronous copies: this is the integration surface, not the fast path
// (cluster.py / the C ABI with device-resident buffers is).
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "demo_b200.h"
#include "demosim/model.hpp"
#include "demosim/optim.hpp"
#include "demosim/replicate.hpp"
#include "demosim/rng.hpp"
#include "demosim/transform.hpp"
#include "demosim/vec.hpp"

namespace demosim {
namespace {

void check(int rc) {
  if (rc == DMB_OK) return;
  const std::string msg = dmb_last_error();
  switch (rc) {
    case DMB_TRAINING: throw TrainingError(msg);
    case DMB_CONFIG: throw ConfigError(msg);
    case DMB_PROTOCOL: throw ProtocolError(msg);
    default: throw std::runtime_error("CUDA: " + msg);
  }
}

dmb_ctx* ctx() {
  static dmb_ctx* c = [] {
    dmb_ctx* h = nullptr;
    check(dmb_ctx_create(0, &h));
    return h;
  }();
  return c;
}

void status() {  // synchronizes; TrainingError / ProtocolError latched on the device
  int64_t bad = -1;
  check(dmb_status(ctx(), nullptr, &bad));
}

// device buffer (RAII)
struct Dev {
  void* p = nullptr;
  explicit Dev(size_t bytes) {
    if (cudaMalloc(&p, bytes ? bytes : 16) != cudaSuccess) throw std::runtime_error("CUDA: cudaMalloc failed");
  }
  ~Dev() { cudaFree(p); }
  Dev(const Dev&) = delete;
  Dev& operator=(const Dev&) = delete;
  float* f() const { return static_cast<float*>(p); }
  uint8_t* b() const { return static_cast<uint8_t*>(p); }
};

std::unique_ptr<Dev> to_device(std::span<const double> v) {
  auto d = std::make_unique<Dev>(v.size() * 4);
  std::vector<float> h(v.begin(), v.end());
  if (!h.empty() && cudaMemcpy(d->p, h.data(), h.size() * 4, cudaMemcpyHostToDevice) != cudaSuccess)
    throw std::runtime_error("CUDA: upload failed");
  return d;
}

DenseVector from_device(const float* d, size_t n) {
  std::vector<float> h(n);
  if (n && cudaMemcpy(h.data(), d, n * 4, cudaMemcpyDeviceToHost) != cudaSuccess)
    throw std::runtime_error("CUDA: download failed");
  return DenseVector(h.begin(), h.end());
}

void into(std::span<double> out, const float* d) {
  const DenseVector h = from_device(d, out.size());
  std::copy(h.begin(), h.end(), out.begin());
}

dmb_rep_cfg cfg_of(const ReplicatorConfig& r) {
  dmb_rep_cfg c{};
  c.scheme = static_cast<int32_t>(r.scheme);
  c.sign_mode = r.sign_mode ? 1 : 0;
  c.transfer_dtype = static_cast<int32_t>(r.transfer_dtype);
  c.chunk_size = r.chunk_size;
  c.top_k = r.top_k;
  c.compression = r.compression;
  c.seed = r.seed;
  return c;
}

dmb_opt_cfg opt_of(const OptimizerConfig& o) {
  dmb_opt_cfg c{};
  c.kind = o.kind == OptimizerKind::DemoSgd ? DMB_DEMO_SGD : DMB_DECOUPLED_ADAMW;
  c.learning_rate = o.learning_rate;
  c.momentum_decay = o.momentum_decay;
  c.adam_beta1 = o.adam_beta1;
  c.adam_beta2 = o.adam_beta2;
  c.adam_eps = o.adam_eps;
  c.weight_decay = o.weight_decay;
  return c;
}

// device update (header + body) -> host CompressedUpdate with values at wire precision
CompressedUpdate to_host(const dmb_update& u, TransferDtype d) {
  CompressedUpdate h;
  h.scheme = static_cast<Scheme>(u.scheme);
  h.step = u.step;
  h.shard_id = u.shard_id;
  h.length = u.length;
  h.empty = u.empty != 0;
  h.chunk_size = u.chunk_size;
  h.top_k = u.top_k;
  h.bytes = u.bytes;
  if (u.n_indices) {
    h.freq_indices.resize(u.n_indices);
    if (cudaMemcpy(h.freq_indices.data(), u.body, u.n_indices * 4, cudaMemcpyDeviceToHost) != cudaSuccess)
      throw std::runtime_error("CUDA: download failed");
  }
  if (u.n_values) {
    Dev vals(u.n_values * 4);
    check(dmb_update_values(&u, static_cast<int32_t>(d), vals.f(), nullptr));
    h.values = from_device(vals.f(), u.n_values);
  }
  return h;
}

// host CompressedUpdate -> the reference body (replicate.cpp:316-356) on the device
struct DevUpdate {
  std::unique_ptr<Dev> body;
  dmb_update u{};
};
DevUpdate to_device(const CompressedUpdate& h, TransferDtype d) {
  std::vector<uint8_t> bytes;
  const size_t ni = h.scheme == Scheme::DeMo ? h.freq_indices.size() : 0;
  for (size_t i = 0; i < ni; ++i)
    for (int k = 0; k < 4; ++k) bytes.push_back(static_cast<uint8_t>(h.freq_indices[i] >> (8 * k)));
  const size_t nv = h.values.size();
  if (d == TransferDtype::Fp32) {
    for (size_t i = 0; i < nv; ++i) {
      const float f = static_cast<float>(h.values[i]);
      uint8_t b[4];
      std::memcpy(b, &f, 4);
      bytes.insert(bytes.end(), b, b + 4);
    }
  } else if (d == TransferDtype::Fp16) {
    for (size_t i = 0; i < nv; ++i) {
      const __half_raw r = __float2half_rn(static_cast<float>(narrow_to_fp16(h.values[i])));
      bytes.push_back(static_cast<uint8_t>(r.x & 0xff));
      bytes.push_back(static_cast<uint8_t>(r.x >> 8));
    }
  } else {
    const size_t base = bytes.size();
    bytes.resize(base + (nv * 2 + 7) / 8, 0);
    for (size_t i = 0; i < nv; ++i) {
      const double v = h.values[i];
      const uint8_t code = v > 0.0 ? 1 : (v < 0.0 ? 2 : 0);
      bytes[base + i / 4] |= static_cast<uint8_t>(code << (2 * (i % 4)));
    }
  }
  DevUpdate out;
  out.body = std::make_unique<Dev>(bytes.size() + 16);
  if (!bytes.empty() && cudaMemcpy(out.body->p, bytes.data(), bytes.size(), cudaMemcpyHostToDevice) != cudaSuccess)
    throw std::runtime_error("CUDA: upload failed");
  out.u.scheme = static_cast<int32_t>(h.scheme);
  out.u.empty = h.empty ? 1 : 0;
  out.u.step = h.step;
  out.u.shard_id = h.shard_id;
  out.u.wire_format = DMB_WIRE_REFERENCE;
  out.u.length = h.length;
  out.u.chunk_size = h.chunk_size;
  out.u.top_k = h.top_k;
  out.u.n_values = nv;
  out.u.n_indices = ni;
  out.u.bytes = h.bytes;
  out.u.body = out.body->p;
  return out;
}

}  // namespace

// ---- rng.hpp -------------------------------------------------------------------------
namespace {
uint64_t finalize(uint64_t z) {  // the splitmix64 finalizer (rng.cpp:10-16)
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
}  // namespace
uint64_t mix_seed(uint64_t seed) { return finalize(seed); }
uint64_t mix_seed(uint64_t seed, uint64_t tag) { return finalize(finalize(seed) ^ tag); }
uint64_t mix_seed(uint64_t seed, uint64_t a, uint64_t b) { return finalize(finalize(finalize(seed) ^ a) ^ b); }

uint64_t Rng::below(uint64_t n) {
  const uint64_t threshold = (0 - n) % n;  // reject the low tail of the 128-bit product
  while (true) {
    const __uint128_t wide = static_cast<__uint128_t>(next_u64()) * n;
    if (static_cast<uint64_t>(wide) >= threshold) return static_cast<uint64_t>(wide >> 64);
  }
}

double Rng::normal() {
  if (have_spare_) {
    have_spare_ = false;
    return spare_;
  }
  const double u1 = 1.0 - uniform();
  const double u2 = uniform();
  const double r = std::sqrt(-2.0 * std::log(u1));
  const double a = 6.283185307179586476925286766559 * u2;
  spare_ = r * std::sin(a);
  have_spare_ = true;
  return r * std::cos(a);
}

// ---- vec.hpp ---------------------------------------------------------------------------
void require_finite(std::span<const double> v, const std::string& what) {
  if (v.empty()) return;
  auto d = to_device(v);
  check(dmb_require_finite(ctx(), d->f(), v.size(), nullptr));
  int64_t bad = -1;
  if (dmb_status(ctx(), nullptr, &bad) == DMB_TRAINING)
    throw TrainingError(what + " contains a non-finite value at index " + std::to_string(bad));
}

DenseVector mean_of(std::span<const DenseVector> vs) {
  if (vs.empty()) throw ProtocolError("mean of an empty set of vectors");
  const size_t n = vs[0].size();
  std::vector<std::unique_ptr<Dev>> ds;
  std::vector<const float*> ptrs;
  for (const DenseVector& v : vs) {
    if (v.size() != n) throw ProtocolError("vectors of different lengths");
    ds.push_back(to_device(v));
    ptrs.push_back(ds.back()->f());
  }
  Dev out(n * 4);
  check(dmb_grad_mean(ctx(), ptrs.data(), ptrs.size(), n, out.f(), nullptr));
  return from_device(out.f(), n);
}

// ---- transform.hpp ---------------------------------------------------------------------
ChunkLayout chunk_layout(std::size_t length, std::size_t chunk_size) {
  dmb_layout l{};
  check(dmb_chunk_layout(length, chunk_size, &l));
  return ChunkLayout{l.length, l.chunk_size, l.num_chunks, l.pad};
}

static dmb_layout layout_of(const ChunkLayout& l) { return dmb_layout{l.length, l.chunk_size, l.num_chunks, l.pad}; }

std::vector<double> chunk(std::span<const double> v, const ChunkLayout& layout) {
  if (v.size() != layout.length) throw ConfigError("chunk: layout does not match the vector");
  auto d = to_device(v);
  Dev rows(layout.num_chunks * layout.chunk_size * 4);
  const dmb_layout l = layout_of(layout);
  check(dmb_chunk(ctx(), d->f(), &l, rows.f(), nullptr));
  return from_device(rows.f(), layout.num_chunks * layout.chunk_size);
}

std::vector<double> unchunk(std::span<const double> rows, const ChunkLayout& layout) {
  if (rows.size() != layout.num_chunks * layout.chunk_size)
    throw ConfigError("unchunk: row buffer does not match the layout");
  auto d = to_device(rows);
  Dev v(layout.length * 4);
  const dmb_layout l = layout_of(layout);
  check(dmb_unchunk(ctx(), d->f(), &l, v.f(), nullptr));
  return from_device(v.f(), layout.length);
}

DctPlan::DctPlan(std::size_t size) : size_(size) {
  if (size == 0) throw ConfigError("transform size must be positive");
  if (size > 1024) throw ConfigError("transform size above the device limit 1024");
}

void DctPlan::forward(std::span<const double> x, std::span<double> out) const {
  auto d = to_device(x.first(size_));
  Dev o(size_ * 4);
  check(dmb_dct2(ctx(), d->f(), size_, 1, o.f(), nullptr));
  into(out.first(size_), o.f());
}

void DctPlan::inverse(std::span<const double> coeffs, std::span<double> out) const {
  auto d = to_device(coeffs.first(size_));
  Dev o(size_ * 4);
  check(dmb_idct3(ctx(), d->f(), size_, 1, o.f(), nullptr));
  into(out.first(size_), o.f());
}

const DctPlan& dct_plan(std::size_t size) {
  thread_local std::map<std::size_t, DctPlan> cache;  // transform.cpp:75-80
  auto it = cache.find(size);
  if (it == cache.end()) it = cache.emplace(size, DctPlan(size)).first;
  return it->second;
}

std::vector<double> dct2(std::span<const double> x) {
  std::vector<double> out(x.size());
  dct_plan(x.size()).forward(x, out);
  return out;
}

std::vector<double> idct3(std::span<const double> coeffs) {
  std::vector<double> out(coeffs.size());
  dct_plan(coeffs.size()).inverse(coeffs, out);
  return out;
}

Extraction extract_fast_components(std::span<const double> v, std::size_t chunk_size, std::size_t top_k) {
  if (top_k == 0 || top_k > chunk_size)
    throw ConfigError("top_k " + std::to_string(top_k) + " out of range for chunk size " + std::to_string(chunk_size));
  Extraction ex;
  ex.selection.layout = chunk_layout(v.size(), chunk_size);
  ex.selection.top_k = top_k;
  const size_t n = ex.selection.layout.num_chunks * top_k;
  auto d = to_device(v);
  Dev idx(n * 4), co(n * 4), fast(v.size() * 4), res(v.size() * 4);
  check(dmb_extract_fast_components(ctx(), d->f(), v.size(), chunk_size, top_k, static_cast<uint32_t*>(idx.p),
                                    co.f(), fast.f(), res.f(), nullptr));
  ex.selection.indices.resize(n);
  if (n && cudaMemcpy(ex.selection.indices.data(), idx.p, n * 4, cudaMemcpyDeviceToHost) != cudaSuccess)
    throw std::runtime_error("CUDA: download failed");
  ex.selection.coeffs = from_device(co.f(), n);
  ex.fast = from_device(fast.f(), v.size());
  ex.residual = from_device(res.f(), v.size());
  return ex;
}

void sign_transform(std::span<double> v) {
  if (v.empty()) return;
  auto d = to_device(v);
  check(dmb_sign_transform(ctx(), d->f(), v.size(), nullptr));
  into(v, d->f());
}

// ---- replicate.hpp ---------------------------------------------------------------------
std::string scheme_name(Scheme s) {
  switch (s) {
    case Scheme::DeMo: return "demo";
    case Scheme::Random: return "random";
    case Scheme::Striding: return "striding";
    case Scheme::DiLoCo: return "diloco";
    case Scheme::Full: return "full";
  }
  return "unknown";
}

std::string dtype_name(TransferDtype d) {
  switch (d) {
    case TransferDtype::Fp32: return "fp32";
    case TransferDtype::Fp16: return "fp16";
    case TransferDtype::Ternary: return "ternary";
  }
  return "unknown";
}

std::size_t value_bits(TransferDtype d) { return d == TransferDtype::Fp16 ? 16 : (d == TransferDtype::Ternary ? 2 : 32); }

uint64_t wire_bytes(std::size_t n_values, std::size_t n_indices, TransferDtype d) {
  return dmb_wire_bytes(n_values, n_indices, static_cast<int32_t>(d));
}

std::size_t ReplicatorConfig::period() const { return dmb_period(compression); }

double narrow_to_fp32(double x) {  // round to nearest even through binary32
  if (std::isnan(x)) return x;
  return static_cast<double>(static_cast<float>(x));  // the conversion is RNE with overflow to inf
}

double narrow_to_fp16(double x) {  // round to nearest even through binary16, from the double
  if (std::isnan(x) || x == 0.0) return x;
  const double a = std::fabs(x), sign = std::signbit(x) ? -1.0 : 1.0;
  const double inf = std::numeric_limits<double>::infinity();
  if (a >= 65520.0) return sign * inf;  // at or beyond the rounding boundary of the largest normal
  int e;
  std::frexp(a, &e);
  const double ulp = std::ldexp(1.0, (e - 1 >= -14 ? e - 1 : -14) - 10);
  const double r = std::nearbyint(a / ulp) * ulp;
  return r >= 65520.0 ? sign * inf : sign * r;
}

EncodeResult select_and_encode(std::span<const double> v, const ReplicatorConfig& cfg, uint64_t step,
                               uint32_t shard_id) {
  const dmb_rep_cfg c = cfg_of(cfg);
  auto d = to_device(v);
  Dev body(dmb_update_capacity(&c, v.size())), lq(v.size() * 4);
  dmb_update u{};
  u.body = body.p;
  check(dmb_select_and_encode(ctx(), d->f(), v.size(), &c, step, shard_id, &u, lq.f(), nullptr));
  EncodeResult r;
  r.update = to_host(u, cfg.transfer_dtype);
  r.local_q = from_device(lq.f(), v.size());
  return r;
}

std::vector<uint32_t> selected_indices(const ReplicatorConfig& cfg, uint64_t step, uint32_t shard_id,
                                       std::size_t length) {
  const dmb_rep_cfg c = cfg_of(cfg);
  Dev out(length * 4);
  uint64_t n = 0;
  check(dmb_selected_indices(ctx(), &c, step, shard_id, length, static_cast<uint32_t*>(out.p), &n, nullptr));
  std::vector<uint32_t> idx(n);
  if (n && cudaMemcpy(idx.data(), out.p, n * 4, cudaMemcpyDeviceToHost) != cudaSuccess)
    throw std::runtime_error("CUDA: download failed");
  return idx;
}

DenseVector decode_and_merge(std::span<const CompressedUpdate> updates, const ReplicatorConfig& cfg) {
  const dmb_rep_cfg c = cfg_of(cfg);
  std::vector<DevUpdate> dev;
  std::vector<dmb_update> ups;
  for (const CompressedUpdate& u : updates) {
    dev.push_back(to_device(u, cfg.transfer_dtype));
    ups.push_back(dev.back().u);
  }
  const size_t n = updates.empty() ? 0 : updates[0].length;
  Dev q(n * 4);
  check(dmb_decode_and_merge(ctx(), ups.data(), ups.size(), &c, q.f(), nullptr));
  return from_device(q.f(), n);
}

std::vector<std::byte> serialize(const CompressedUpdate& u, TransferDtype d) {
  DevUpdate du = to_device(u, d);
  du.u.bytes = dmb_wire_bytes(du.u.n_values, du.u.n_indices, static_cast<int32_t>(d));
  std::vector<uint8_t> buf(9 + du.u.bytes + 16);
  uint64_t written = 0;
  check(dmb_serialize(&du.u, static_cast<int32_t>(d), buf.data(), buf.size(), &written, nullptr));
  std::vector<std::byte> out(written);
  std::memcpy(out.data(), buf.data(), written);
  return out;
}

CompressedUpdate deserialize(std::span<const std::byte> buf, TransferDtype d, const CompressedUpdate& shape_template) {
  DevUpdate tmpl = to_device(shape_template, d);
  Dev body(buf.size() + 16);
  dmb_update out{};
  out.body = body.p;
  check(dmb_deserialize(reinterpret_cast<const uint8_t*>(buf.data()), buf.size(), static_cast<int32_t>(d), &tmpl.u,
                        &out, nullptr));
  return to_host(out, d);
}

// ---- optim.hpp -------------------------------------------------------------------------
MomentumState MomentumState::make(OptimizerKind kind, std::size_t len) {
  MomentumState st;
  if (kind == OptimizerKind::DemoSgd) st.m.assign(len, 0.0);
  else {
    st.exp_avg.assign(len, 0.0);
    st.exp_avg_sq.assign(len, 0.0);
  }
  return st;
}

EncodeResult demo_sgd_prepare(MomentumState& state, std::span<const double> grad, const OptimizerConfig& opt,
                              const ReplicatorConfig& rep, uint64_t step, uint32_t shard_id, StepTrace* trace) {
  require_finite(grad, "gradient");  // before the length check, as optim.cpp:21-24
  if (grad.size() != state.m.size()) throw ProtocolError("gradient and momentum lengths disagree");
  const size_t n = grad.size();
  const dmb_rep_cfg c = cfg_of(rep);
  const dmb_opt_cfg o = opt_of(opt);
  auto g = to_device(grad), m = to_device(state.m);
  Dev m_out(n * 4), lq(n * 4), acc(n * 4), body(dmb_update_capacity(&c, n));
  dmb_update u{};
  u.body = body.p;
  check(dmb_demo_sgd_prepare(ctx(), g->f(), m->f(), m_out.f(), n, &o, &c, step, shard_id, &u, lq.f(), acc.f(),
                             nullptr));
  status();  // a refused step leaves state.m as it was
  EncodeResult r;
  r.update = to_host(u, rep.transfer_dtype);
  r.local_q = from_device(lq.f(), n);
  state.m = from_device(m_out.f(), n);
  if (trace) {
    trace->m_accum = from_device(acc.f(), n);
    trace->local_q = r.local_q;
    trace->m_after = state.m;
  }
  return r;
}

void demo_sgd_apply(std::span<double> params, std::span<const double> q, double lr) {
  auto p = to_device(params), dq = to_device(q);
  check(dmb_demo_sgd_apply(ctx(), p->f(), dq->f(), params.size(), lr, nullptr));
  status();
  into(params, p->f());
}

EncodeResult adamw_prepare(std::span<const double> grad, const ReplicatorConfig& rep, uint64_t step,
                           uint32_t shard_id) {
  require_finite(grad, "gradient");
  const size_t n = grad.size();
  const dmb_rep_cfg c = cfg_of(rep);
  auto g = to_device(grad);
  Dev lq(n * 4), body(dmb_update_capacity(&c, n));
  dmb_update u{};
  u.body = body.p;
  check(dmb_adamw_prepare(ctx(), g->f(), n, &c, step, shard_id, &u, lq.f(), nullptr));
  status();
  EncodeResult r;
  r.update = to_host(u, rep.transfer_dtype);
  r.local_q = from_device(lq.f(), n);
  return r;
}

void adamw_apply(std::span<double> params, MomentumState& state, std::span<const double> grad,
                 std::span<const double> local_q, const DenseVector* merged, const OptimizerConfig& opt, double lr) {
  const size_t n = params.size();
  const dmb_opt_cfg o = opt_of(opt);
  auto p = to_device(params), ea = to_device(state.exp_avg), es = to_device(state.exp_avg_sq);
  auto g = to_device(grad), lq = to_device(local_q);
  std::unique_ptr<Dev> mg = merged ? to_device(*merged) : nullptr;
  uint64_t steps = state.steps;
  check(dmb_adamw_apply(ctx(), p->f(), ea->f(), es->f(), &steps, g->f(), lq->f(), mg ? mg->f() : nullptr, n, &o, lr,
                        nullptr));
  status();
  state.steps = steps;
  into(params, p->f());
  state.exp_avg = from_device(ea->f(), n);
  state.exp_avg_sq = from_device(es->f(), n);
}

void baseline_sgd_step(std::span<double> params, MomentumState& state, std::span<const double> grad,
                       const OptimizerConfig& opt, double lr) {
  require_finite(grad, "gradient");
  const dmb_opt_cfg o = opt_of(opt);
  auto p = to_device(params), m = to_device(state.m), g = to_device(grad);
  check(dmb_baseline_sgd_step(ctx(), p->f(), m->f(), g->f(), params.size(), &o, lr, nullptr));
  status();
  into(params, p->f());
  state.m = from_device(m->f(), state.m.size());
}

void baseline_adamw_step(std::span<double> params, MomentumState& state, std::span<const double> grad,
                         const OptimizerConfig& opt, double lr) {
  require_finite(grad, "gradient");  // optim.cpp:88-93: adamw_apply(params, state, grad, grad, nullptr)
  adamw_apply(params, state, grad, grad, nullptr, opt, lr);
}

// ---- model.hpp (model.cpp:121-244): the toy producers on the device -----------------------------
// loss and gradient of a host batch by dmb_toy_loss_grad / dmb_toy_loss: the batch becomes the
// pool (identity order, one worker), parameters go to the device as FP32 and the FP64 loss and
// the FP32 gradient come back; init_params draws on the host (the reference's Rng)
std::size_t Model::param_count() const {  // model.cpp:121-125
  if (kind == ModelKind::Quadratic) return layer_dims.front();
  std::size_t total = 0;
  for (std::size_t l = 0; l + 1 < layer_dims.size(); ++l) total += layer_dims[l + 1] * layer_dims[l] + layer_dims[l + 1];
  return total;
}

static void check_batch(const Model& model, std::span<const double> params, const Batch& batch) {  // model.cpp:13-35
  char buf[160];
  if (params.size() < model.param_count()) {
    std::snprintf(buf, sizeof buf, "parameter vector too short: %zu < %zu", params.size(), model.param_count());
    throw ConfigError(buf);
  }
  if (batch.size == 0) throw ConfigError("empty batch");
  if (batch.input_dim != model.input_dim()) {
    std::snprintf(buf, sizeof buf, "batch input dim %zu does not match model input dim %zu", batch.input_dim,
                  model.input_dim());
    throw ConfigError(buf);
  }
  if (model.kind == ModelKind::Mlp) {
    if (model.loss == LossKind::CrossEntropy) {
      if (batch.labels.size() != batch.size) throw ConfigError("cross entropy batch is missing labels");
    } else if (batch.targets.size() != batch.size * model.output_dim()) {
      throw ConfigError("regression batch targets do not match model output dim");
    }
  }
  if (model.layer_dims.size() > 9) throw ConfigError("the device producer takes at most 8 layers");
}

namespace {
struct DevBatch {  // a host batch as a device pool
  std::unique_ptr<Dev> in, tgt, lab;
  dmb_toy_pool pool{};
  DevBatch(const Model& m, const Batch& b) {
    auto put = [](const void* src, size_t bytes) {
      auto d = std::make_unique<Dev>(bytes);
      if (bytes && cudaMemcpy(d->p, src, bytes, cudaMemcpyHostToDevice) != cudaSuccess)
        throw std::runtime_error("CUDA: upload failed");
      return d;
    };
    in = put(b.inputs.data(), b.size * b.input_dim * 8);
    pool.inputs = static_cast<const double*>(in->p);
    if (m.kind == ModelKind::Mlp && m.loss == LossKind::Mse) {
      tgt = put(b.targets.data(), b.targets.size() * 8);
      pool.targets = static_cast<const double*>(tgt->p);
    }
    if (m.kind == ModelKind::Mlp && m.loss == LossKind::CrossEntropy) {
      std::vector<int32_t> l(b.labels.begin(), b.labels.end());
      lab = put(l.data(), l.size() * 4);
      pool.labels = static_cast<const int32_t*>(lab->p);
    }
    pool.size = b.size;
  }
};
dmb_toy_model toy_of(const Model& m) {
  dmb_toy_model t{};
  t.kind = m.kind == ModelKind::Quadratic ? 0u : 1u;
  t.activation = m.activation == Activation::Tanh ? 0u : 1u;
  t.loss = m.loss == LossKind::Mse ? 0u : 1u;
  t.n_dims = (uint32_t)m.layer_dims.size();
  for (size_t l = 0; l < m.layer_dims.size(); ++l) t.dims[l] = (uint32_t)m.layer_dims[l];
  return t;
}
double loss_of(const Dev& loss) {
  double h = 0.0;
  if (cudaMemcpy(&h, loss.p, 8, cudaMemcpyDeviceToHost) != cudaSuccess) throw std::runtime_error("CUDA: download failed");
  return h;
}
}  // namespace

double forward_loss(const Model& model, std::span<const double> params, const Batch& batch) {
  check_batch(model, params, batch);
  const dmb_toy_model t = toy_of(model);
  DevBatch db(model, batch);
  auto p = to_device(params.first(model.param_count()));
  Dev loss(8);
  check(dmb_toy_loss(ctx(), &t, &db.pool, p->f(), static_cast<double*>(loss.p), nullptr));
  status();
  return loss_of(loss);
}

LossAndGradient loss_and_gradient(const Model& model, std::span<const double> params, const Batch& batch) {
  check_batch(model, params, batch);
  const dmb_toy_model t = toy_of(model);
  DevBatch db(model, batch);
  auto p = to_device(params);
  std::vector<int64_t> order(batch.size);
  for (size_t i = 0; i < batch.size; ++i) order[i] = (int64_t)i;
  Dev dord(order.size() * 8), g(params.size() * 4), loss(8);
  if (cudaMemcpy(dord.p, order.data(), order.size() * 8, cudaMemcpyHostToDevice) != cudaSuccess)
    throw std::runtime_error("CUDA: upload failed");
  check(dmb_toy_loss_grad(ctx(), &t, &db.pool, static_cast<const int64_t*>(dord.p), 0, batch.size, p->f(),
                          params.size(), 1, 1, g.f(), params.size(), static_cast<double*>(loss.p), nullptr));
  status();
  LossAndGradient r;
  r.loss = loss_of(loss);
  r.grad = from_device(g.f(), params.size());  // the pad tail gets exact zeros
  return r;
}

DenseVector gradient(const Model& model, std::span<const double> params, const Batch& batch) {
  return loss_and_gradient(model, params, batch).grad;
}

DenseVector finite_diff_gradient(const Model& model, std::span<const double> params, const Batch& batch,
                                 double h) {  // model.cpp:209-222
  if (!(h > 0.0)) throw ConfigError("finite difference step must be positive");
  DenseVector theta(params.begin(), params.end());
  DenseVector out(params.size(), 0.0);
  for (size_t i = 0; i < theta.size(); ++i) {
    const double saved = theta[i];
    theta[i] = saved + h;
    const double up = forward_loss(model, theta, batch);
    theta[i] = saved - h;
    const double down = forward_loss(model, theta, batch);
    theta[i] = saved;
    out[i] = (up - down) / (2.0 * h);
  }
  return out;
}

DenseVector init_params(const Model& model, uint64_t seed, std::size_t padded_len) {  // model.cpp:224-244
  const size_t n = model.param_count();
  if (padded_len < n) throw ConfigError("padded parameter length shorter than the model");
  DenseVector params(padded_len, 0.0);
  if (model.kind == ModelKind::Quadratic) return params;
  Rng rng(mix_seed(seed, 0x6d6f64656cULL));
  size_t off = 0;
  for (size_t l = 0; l + 1 < model.layer_dims.size(); ++l) {
    const size_t in = model.layer_dims[l], out = model.layer_dims[l + 1];
    const double bound = 1.0 / std::sqrt(static_cast<double>(in));
    for (size_t k = 0; k < out * in + out; ++k) params[off + k] = rng.uniform(-bound, bound);
    off += out * in + out;
  }
  return params;
}

}  // namespace demosim
