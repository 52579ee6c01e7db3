// ref_shim.cpp -- extern "C" face over the UNMODIFIED reference core.
//
// TEST INFRASTRUCTURE ONLY.  oracle/Makefile compiles this file together with
// the reference's own sources where they lie (/root/reference/proj/core/src/
// {vec,rng,transform,replicate,optim,cluster}.cpp, reference flags -O3, no
// -march) into oracle/_ref/libdemosim_ref.so.  It exports the same dmo_* C
// signatures as the restatement in demo_oracle.c, so tests/ can run both on the
// same inputs and pin the restatement to the reference bit for bit, and bench.py
// can time the reference's own CPU path ("kind": "reference").
#include <cstdint>
#include <cstring>
#include <span>
#include <string>
#include <vector>

#include "demosim/cluster.hpp"
#include "demosim/optim.hpp"
#include "demosim/replicate.hpp"
#include "demosim/rng.hpp"
#include "demosim/transform.hpp"
#include "demosim/vec.hpp"

#include "demo_oracle.h"

namespace demosim {
// cluster.cpp:59 references trainer.cpp's formatter; the ledger CSV writer is
// never called through this shim, so a plain %.17g formatter suffices.
std::string format_double(double x) {
  char buf[40];
  std::snprintf(buf, sizeof buf, "%.17g", x);
  return buf;
}
}  // namespace demosim

using namespace demosim;

namespace {
thread_local std::string g_err;

ReplicatorConfig to_cfg(const dmo_rep_cfg* c) {
  ReplicatorConfig r;
  r.scheme = static_cast<Scheme>(c->scheme);
  r.chunk_size = c->chunk_size;
  r.top_k = c->top_k;
  r.compression = c->compression;
  r.sign_mode = c->sign_mode != 0;
  r.transfer_dtype = static_cast<TransferDtype>(c->transfer_dtype);
  r.seed = c->seed;
  return r;
}

template <typename Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    return DMO_OK;
  } catch (const TrainingError& e) {
    g_err = e.what();
    return DMO_TRAINING;
  } catch (const ConfigError& e) {
    g_err = e.what();
    return DMO_CONFIG;
  } catch (const ProtocolError& e) {
    g_err = e.what();
    return DMO_PROTOCOL;
  }
}

void export_encode(const EncodeResult& enc, uint32_t* freq_indices, double* values,
                   uint64_t* n_values, uint64_t* bytes, int32_t* empty, double* local_q) {
  const CompressedUpdate& u = enc.update;
  if (freq_indices && !u.freq_indices.empty())
    std::memcpy(freq_indices, u.freq_indices.data(), u.freq_indices.size() * 4);
  if (!u.values.empty()) std::memcpy(values, u.values.data(), u.values.size() * 8);
  *n_values = u.values.size();
  *bytes = u.bytes;
  *empty = u.empty ? 1 : 0;
  std::memcpy(local_q, enc.local_q.data(), enc.local_q.size() * 8);
}
}  // namespace

extern "C" {

const char* dmo_last_error(void) { return g_err.c_str(); }

uint64_t dmo_mix_seed1(uint64_t s) { return mix_seed(s); }
uint64_t dmo_mix_seed2(uint64_t s, uint64_t a) { return mix_seed(s, a); }
uint64_t dmo_mix_seed3(uint64_t s, uint64_t a, uint64_t b) { return mix_seed(s, a, b); }

void dmo_random_vector(uint64_t seed, size_t n, double* out) {
  Rng rng(seed);
  for (size_t i = 0; i < n; ++i) out[i] = rng.normal();
}

/* raw std::mt19937_64 stream, for the engine known-answer test */
void dmo_mt64_stream(uint64_t seed, uint64_t n, uint64_t* out) {
  std::mt19937_64 e(seed);
  for (uint64_t i = 0; i < n; ++i) out[i] = e();
}

void dmo_rng_below_batch(uint64_t seed, const uint64_t* ns, uint64_t count, uint64_t* out) {
  Rng rng(seed);
  for (uint64_t i = 0; i < count; ++i) out[i] = rng.below(ns[i]);
}

void dmo_dct_basis(size_t s, double* basis) {
  // The plan keeps its basis private; probe forward() with unit vectors:
  // forward(e_i)[j] = 0.0 + B[j][i]*1.0 + 0*... = B[j][i] exactly.
  const DctPlan& plan = dct_plan(s);
  std::vector<double> e(s, 0.0), out(s);
  for (size_t i = 0; i < s; ++i) {
    std::fill(e.begin(), e.end(), 0.0);
    e[i] = 1.0;
    plan.forward(e, out);
    for (size_t j = 0; j < s; ++j) basis[j * s + i] = out[j];
  }
}

void dmo_dct_forward(size_t s, const double*, const double* x, double* out) {
  dct_plan(s).forward(std::span<const double>(x, s), std::span<double>(out, s));
}
void dmo_dct_inverse(size_t s, const double*, const double* c, double* out) {
  dct_plan(s).inverse(std::span<const double>(c, s), std::span<double>(out, s));
}

int dmo_extract_fast_components(const double* v, size_t len, size_t s, size_t top_k,
                                uint32_t* indices, double* coeffs, double* fast,
                                double* residual) {
  return guarded([&] {
    Extraction ex = extract_fast_components(std::span<const double>(v, len), s, top_k);
    std::memcpy(indices, ex.selection.indices.data(), ex.selection.indices.size() * 4);
    std::memcpy(coeffs, ex.selection.coeffs.data(), ex.selection.coeffs.size() * 8);
    std::memcpy(fast, ex.fast.data(), len * 8);
    if (residual) std::memcpy(residual, ex.residual.data(), len * 8);
  });
}

void dmo_sign_transform(double* v, size_t n) { sign_transform(std::span<double>(v, n)); }
uint64_t dmo_wire_bytes(uint64_t nv, uint64_t ni, int d) {
  return wire_bytes(nv, ni, static_cast<TransferDtype>(d));
}
uint64_t dmo_period(double c) {
  ReplicatorConfig r;
  r.compression = c;
  return r.period();
}
double dmo_narrow_to_fp16(double x) { return narrow_to_fp16(x); }
double dmo_narrow_to_fp32(double x) { return narrow_to_fp32(x); }

int dmo_selected_indices(const dmo_rep_cfg* cfg, uint64_t step, uint32_t shard, uint64_t len,
                         uint32_t* out, uint64_t* count) {
  return guarded([&] {
    const std::vector<uint32_t> idx = selected_indices(to_cfg(cfg), step, shard, len);
    std::memcpy(out, idx.data(), idx.size() * 4);
    *count = idx.size();
  });
}

int dmo_select_and_encode(const double* v, uint64_t len, const dmo_rep_cfg* cfg, uint64_t step,
                          uint32_t shard, uint32_t* freq_indices, double* values,
                          uint64_t* n_values, uint64_t* n_indices, uint64_t* bytes,
                          int32_t* empty, double* local_q) {
  return guarded([&] {
    const EncodeResult enc =
        select_and_encode(std::span<const double>(v, len), to_cfg(cfg), step, shard);
    export_encode(enc, freq_indices, values, n_values, bytes, empty, local_q);
    *n_indices = enc.update.freq_indices.size();
  });
}

int dmo_decode_and_merge(const dmo_rep_cfg* cfg, uint64_t replicas, const double* const* values,
                         const uint32_t* const* freq_indices, uint64_t n_values, uint64_t len,
                         uint64_t step, uint32_t shard, double* q) {
  return guarded([&] {
    const ReplicatorConfig rc = to_cfg(cfg);
    std::vector<CompressedUpdate> ups(replicas);
    for (uint64_t r = 0; r < replicas; ++r) {
      CompressedUpdate& u = ups[r];
      u.scheme = rc.scheme;
      u.step = step;
      u.shard_id = shard;
      u.length = len;
      u.values.assign(values[r], values[r] + n_values);
      if (rc.scheme == Scheme::DeMo) {
        u.chunk_size = rc.chunk_size;
        u.top_k = rc.top_k;
        u.freq_indices.assign(freq_indices[r], freq_indices[r] + n_values);
      }
    }
    const DenseVector out = decode_and_merge(ups, rc);
    std::memcpy(q, out.data(), len * 8);
  });
}

uint64_t dmo_serialize(int scheme, const uint32_t* freq_indices, uint64_t n_indices,
                       const double* values, uint64_t n_values, int dtype, uint8_t* out) {
  CompressedUpdate u;
  u.scheme = static_cast<Scheme>(scheme);
  if (u.scheme == Scheme::DeMo) u.freq_indices.assign(freq_indices, freq_indices + n_indices);
  u.values.assign(values, values + n_values);
  u.bytes = wire_bytes(n_values, u.freq_indices.size(), static_cast<TransferDtype>(dtype));
  const std::vector<std::byte> buf = serialize(u, static_cast<TransferDtype>(dtype));
  std::memcpy(out, buf.data(), buf.size());
  return buf.size();
}

int dmo_demo_sgd_prepare(double* m, const double* grad, uint64_t len, double beta,
                         const dmo_rep_cfg* cfg, uint64_t step, uint32_t shard,
                         uint32_t* freq_indices, double* values, uint64_t* n_values,
                         uint64_t* bytes, int32_t* empty, double* local_q,
                         double* m_accum_trace, int64_t* bad_index) {
  if (bad_index) *bad_index = -1;
  return guarded([&] {
    MomentumState st;
    st.m.assign(m, m + len);
    OptimizerConfig opt;
    opt.momentum_decay = beta;
    StepTrace tr;
    const EncodeResult enc = demo_sgd_prepare(st, std::span<const double>(grad, len), opt,
                                              to_cfg(cfg), step, shard, &tr);
    export_encode(enc, freq_indices, values, n_values, bytes, empty, local_q);
    if (m_accum_trace) std::memcpy(m_accum_trace, tr.m_accum.data(), len * 8);
    std::memcpy(m, st.m.data(), len * 8);
  });
}

void dmo_demo_sgd_apply(double* params, const double* q, uint64_t n, double lr) {
  demo_sgd_apply(std::span<double>(params, n), std::span<const double>(q, n), lr);
}

void dmo_adamw_apply(double* params, double* exp_avg, double* exp_avg_sq, uint64_t* steps,
                     const double* grad, const double* local_q, const double* merged,
                     uint64_t n, double beta1, double beta2, double eps, double weight_decay,
                     double lr) {
  MomentumState st;
  st.exp_avg.assign(exp_avg, exp_avg + n);
  st.exp_avg_sq.assign(exp_avg_sq, exp_avg_sq + n);
  st.steps = *steps;
  OptimizerConfig opt;
  opt.kind = OptimizerKind::DecoupledAdamW;
  opt.adam_beta1 = beta1;
  opt.adam_beta2 = beta2;
  opt.adam_eps = eps;
  opt.weight_decay = weight_decay;
  DenseVector mg;
  if (merged) mg.assign(merged, merged + n);
  adamw_apply(std::span<double>(params, n), st, std::span<const double>(grad, n),
              std::span<const double>(local_q, n), merged ? &mg : nullptr, opt, lr);
  std::memcpy(exp_avg, st.exp_avg.data(), n * 8);
  std::memcpy(exp_avg_sq, st.exp_avg_sq.data(), n * 8);
  *steps = st.steps;
}

int dmo_grad_reduce_scatter(uint64_t members, uint64_t len, const double* const* grads,
                            double* shards) {
  return guarded([&] {
    std::vector<DenseVector> gs(members);
    for (uint64_t a = 0; a < members; ++a) gs[a].assign(grads[a], grads[a] + len);
    const std::vector<DenseVector> out = grad_reduce_scatter(gs, nullptr);
    uint64_t off = 0;
    for (const DenseVector& s : out) {
      std::memcpy(shards + off, s.data(), s.size() * 8);
      off += s.size();
    }
  });
}

}  // extern "C"
