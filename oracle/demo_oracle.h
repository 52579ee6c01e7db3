/*
 * demo_oracle.h -- CPU restatement of the demosim FlexDeMo optimizer-step path.
 *
 * TEST INFRASTRUCTURE ONLY.  This is the checker the CUDA product path is
 * compared against; it is never linked into, loaded by, or called from the
 * product library (paper_2502_06728_b200/).  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg may use it.
 *
 * Plain C11, FP64, scalar, single threaded.  Every function restates one
 * function of the reference (/root/reference/proj/core, cited file:line) with
 * the same operation order, so results are bit-identical to the reference when
 * compiled without FMA contraction (-ffp-contract=off, no -march), which is how
 * the reference itself is built (proj/CMakeLists.txt:4-8).
 *
 * Pinning: checked against (1) the literal known answers in the reference's own
 * tests (tests/test_oracle_golden.py) and (2) golden vectors produced by the
 * reference compiled unchanged from /root/reference (oracle/Makefile target
 * _ref, generator oracle/gen_golden.py, fixtures tests/golden/).
 */
#ifndef DEMO_ORACLE_H
#define DEMO_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* error codes follow common.hpp:10-26 (ConfigError/ProtocolError/TrainingError) */
enum { DMO_OK = 0, DMO_TRAINING = 1, DMO_CONFIG = 2, DMO_PROTOCOL = 3 };
/* replicate.hpp:14 wire tags */
enum { DMO_DEMO = 1, DMO_RANDOM = 2, DMO_STRIDING = 3, DMO_DILOCO = 4, DMO_FULL = 5 };
/* replicate.hpp:16 */
enum { DMO_FP32 = 0, DMO_FP16 = 1, DMO_TERNARY = 2 };

const char* dmo_last_error(void);

/* ---- rng.hpp / rng.cpp ------------------------------------------------- */
uint64_t dmo_mix64(uint64_t z);
uint64_t dmo_mix_seed1(uint64_t seed);
uint64_t dmo_mix_seed2(uint64_t seed, uint64_t tag);
uint64_t dmo_mix_seed3(uint64_t seed, uint64_t tag_a, uint64_t tag_b);

typedef struct {
  uint64_t mt[312];
  int idx;
} dmo_mt64;
void dmo_mt64_seed(dmo_mt64* e, uint64_t seed);
uint64_t dmo_mt64_next(dmo_mt64* e);

typedef struct {
  dmo_mt64 eng;
  int have_spare;
  double spare;
} dmo_rng;
void dmo_rng_init(dmo_rng* r, uint64_t seed);
uint64_t dmo_rng_next_u64(dmo_rng* r);
double dmo_rng_uniform(dmo_rng* r);
uint64_t dmo_rng_below(dmo_rng* r, uint64_t n);
double dmo_rng_normal(dmo_rng* r);
/* raw engine stream (KAT) and batched below() draws from Rng(seed) */
void dmo_mt64_stream(uint64_t seed, uint64_t n, uint64_t* out);
void dmo_rng_below_batch(uint64_t seed, const uint64_t* ns, uint64_t count, uint64_t* out);
/* the reference tests' random_vector(seed, n) helper (test_transform.cpp:18-23) */
void dmo_random_vector(uint64_t seed, size_t n, double* out);

/* ---- transform.hpp / transform.cpp --------------------------------------- */
size_t dmo_num_chunks(size_t length, size_t chunk_size);
void dmo_dct_basis(size_t s, double* basis /* s*s, basis[j*s+i] */);
void dmo_dct_forward(size_t s, const double* basis, const double* x, double* out);
void dmo_dct_inverse(size_t s, const double* basis, const double* coeffs, double* out);
int dmo_extract_fast_components(const double* v, size_t len, size_t s, size_t top_k,
                                uint32_t* indices /* C*k */, double* coeffs /* C*k */,
                                double* fast /* len */, double* residual /* len or NULL */);
void dmo_sign_transform(double* v, size_t n);

/* ---- replicate.hpp / replicate.cpp --------------------------------------- */
typedef struct {
  int32_t scheme;
  int32_t sign_mode;
  int32_t transfer_dtype;
  int32_t _pad;
  uint64_t chunk_size;
  uint64_t top_k;
  double compression;
  uint64_t seed;
} dmo_rep_cfg;

size_t dmo_value_bits(int dtype);
uint64_t dmo_wire_bytes(uint64_t n_values, uint64_t n_indices, int dtype);
uint64_t dmo_period(double compression);
double dmo_narrow_to_fp16(double x);
double dmo_narrow_to_fp32(double x);
uint16_t dmo_fp16_bits(double x);
/* number of values select_and_encode transmits for this cfg/step/len; -1 + error on config error */
int64_t dmo_value_count(const dmo_rep_cfg* cfg, uint64_t step, uint64_t len);
int dmo_selected_indices(const dmo_rep_cfg* cfg, uint64_t step, uint32_t shard, uint64_t len,
                         uint32_t* out, uint64_t* count);
/* outputs sized by dmo_value_count; freq_indices only written for DeMo */
int dmo_select_and_encode(const double* v, uint64_t len, const dmo_rep_cfg* cfg, uint64_t step,
                          uint32_t shard, uint32_t* freq_indices, double* values,
                          uint64_t* n_values, uint64_t* n_indices, uint64_t* bytes,
                          int32_t* empty, double* local_q);
/* values: R arrays of n_values each (rank order); freq_indices: R arrays (DeMo only) */
int dmo_decode_and_merge(const dmo_rep_cfg* cfg, uint64_t replicas, const double* const* values,
                         const uint32_t* const* freq_indices, uint64_t n_values, uint64_t len,
                         uint64_t step, uint32_t shard, double* q);
/* body of serialize() without/with the 9-byte header; returns bytes written */
uint64_t dmo_serialize(int scheme, const uint32_t* freq_indices, uint64_t n_indices,
                       const double* values, uint64_t n_values, int dtype, uint8_t* out);

/* ---- optim.hpp / optim.cpp ---------------------------------------------- */
int dmo_demo_sgd_prepare(double* m, const double* grad, uint64_t len, double beta,
                         const dmo_rep_cfg* cfg, uint64_t step, uint32_t shard,
                         uint32_t* freq_indices, double* values, uint64_t* n_values,
                         uint64_t* bytes, int32_t* empty, double* local_q,
                         double* m_accum_trace /* nullable */, int64_t* bad_index);
void dmo_demo_sgd_apply(double* params, const double* q, uint64_t n, double lr);
void dmo_adamw_apply(double* params, double* exp_avg, double* exp_avg_sq, uint64_t* steps,
                     const double* grad, const double* local_q, const double* merged /*nullable*/,
                     uint64_t n, double beta1, double beta2, double eps, double weight_decay,
                     double lr);
int dmo_baseline_sgd_step(double* params, double* m, const double* grad, uint64_t n,
                          double beta, double lr);
int dmo_baseline_adamw_step(double* params, double* exp_avg, double* exp_avg_sq, uint64_t* steps,
                            const double* grad, uint64_t n, double beta1, double beta2,
                            double eps, double weight_decay, double lr);
int64_t dmo_first_nonfinite(const double* v, uint64_t n);

/* ---- cluster.cpp:63-91 --------------------------------------------------- */
int dmo_grad_reduce_scatter(uint64_t members, uint64_t len, const double* const* grads,
                            double* shards /* members x (len/members) */);

#ifdef __cplusplus
}
#endif
#endif
