/*
 * demo_oracle.c -- FP64 CPU restatement of the demosim optimizer-step path.
 *
 * TEST INFRASTRUCTURE ONLY (see demo_oracle.h).  Build: oracle/Makefile
 * (gcc -O2 -ffp-contract=off, no -march, like the reference's own flags).
 */
#define _GNU_SOURCE
#include "demo_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static char g_err[256];

const char* dmo_last_error(void) { return g_err; }

static int fail(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}

/* ======================= rng.cpp ======================================== */

/* splitmix64 finalizer, rng.cpp:10-15 */
uint64_t dmo_mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
/* rng.cpp:19-25 */
uint64_t dmo_mix_seed1(uint64_t seed) { return dmo_mix64(seed); }
uint64_t dmo_mix_seed2(uint64_t seed, uint64_t tag) { return dmo_mix64(dmo_mix64(seed) ^ tag); }
uint64_t dmo_mix_seed3(uint64_t seed, uint64_t a, uint64_t b) {
  return dmo_mix64(dmo_mix64(dmo_mix64(seed) ^ a) ^ b);
}

/* std::mt19937_64 as pinned by [rand.predef]: w=64 n=312 m=156 r=31,
 * a=0xb5026f5aa96619e9 u=29 d=0x5555555555555555 s=17 b=0x71d67fffeda60000
 * t=37 c=0xfff7eee000000000 l=43 f=6364136223846793005 (rng.hpp:48). */
void dmo_mt64_seed(dmo_mt64* e, uint64_t seed) {
  e->mt[0] = seed;
  for (int i = 1; i < 312; ++i) {
    e->mt[i] = 6364136223846793005ULL * (e->mt[i - 1] ^ (e->mt[i - 1] >> 62)) + (uint64_t)i;
  }
  e->idx = 312;
}

uint64_t dmo_mt64_next(dmo_mt64* e) {
  const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
  if (e->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      uint64_t x = (e->mt[i] & UM) | (e->mt[(i + 1) % 312] & LM);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
      e->mt[i] = e->mt[(i + 156) % 312] ^ xa;
    }
    e->idx = 0;
  }
  uint64_t y = e->mt[e->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

/* Rng(seed): engine seeded with mix_seed(seed), rng.hpp:21 */
void dmo_rng_init(dmo_rng* r, uint64_t seed) {
  dmo_mt64_seed(&r->eng, dmo_mix_seed1(seed));
  r->have_spare = 0;
  r->spare = 0.0;
}
uint64_t dmo_rng_next_u64(dmo_rng* r) { return dmo_mt64_next(&r->eng); }
/* rng.hpp:26 */
double dmo_rng_uniform(dmo_rng* r) { return (double)(dmo_rng_next_u64(r) >> 11) * 0x1.0p-53; }

/* Lemire debiased multiply-shift, rng.cpp:27-37 */
uint64_t dmo_rng_below(dmo_rng* r, uint64_t n) {
  const uint64_t threshold = (0 - n) % n;
  for (;;) {
    const uint64_t x = dmo_rng_next_u64(r);
    const unsigned __int128 wide = (unsigned __int128)x * n;
    if ((uint64_t)wide >= threshold) return (uint64_t)(wide >> 64);
  }
}

/* Box-Muller with cached spare, rng.cpp:39-51 */
double dmo_rng_normal(dmo_rng* r) {
  if (r->have_spare) {
    r->have_spare = 0;
    return r->spare;
  }
  const double u1 = 1.0 - dmo_rng_uniform(r);
  const double u2 = dmo_rng_uniform(r);
  const double rr = sqrt(-2.0 * log(u1));
  const double a = 6.283185307179586476925286766559 * u2;
  r->spare = rr * sin(a);
  r->have_spare = 1;
  return rr * cos(a);
}

void dmo_mt64_stream(uint64_t seed, uint64_t n, uint64_t* out) {
  dmo_mt64 e;
  dmo_mt64_seed(&e, seed);
  for (uint64_t i = 0; i < n; ++i) out[i] = dmo_mt64_next(&e);
}

void dmo_rng_below_batch(uint64_t seed, const uint64_t* ns, uint64_t count, uint64_t* out) {
  dmo_rng r;
  dmo_rng_init(&r, seed);
  for (uint64_t i = 0; i < count; ++i) out[i] = dmo_rng_below(&r, ns[i]);
}

void dmo_random_vector(uint64_t seed, size_t n, double* out) {
  dmo_rng r;
  dmo_rng_init(&r, seed);
  for (size_t i = 0; i < n; ++i) out[i] = dmo_rng_normal(&r);
}

/* ======================= transform.cpp ================================== */

static const double kPi = 3.14159265358979323846264338327950288;

/* transform.cpp:17-25 */
size_t dmo_num_chunks(size_t length, size_t chunk_size) {
  return (length + chunk_size - 1) / chunk_size;
}

/* DctPlan ctor, transform.cpp:41-54 (same expression order, libm cos) */
void dmo_dct_basis(size_t s, double* basis) {
  const double n = (double)s;
  const double c0 = sqrt(1.0 / n);
  const double cj = sqrt(2.0 / n);
  for (size_t j = 0; j < s; ++j) {
    const double scale = j == 0 ? c0 : cj;
    for (size_t i = 0; i < s; ++i) {
      basis[j * s + i] = scale * cos(kPi * (2.0 * (double)i + 1.0) * (double)j / (2.0 * n));
    }
  }
}

/* DctPlan::forward, transform.cpp:56-63: ascending i from 0.0 */
void dmo_dct_forward(size_t s, const double* basis, const double* x, double* out) {
  for (size_t j = 0; j < s; ++j) {
    const double* row = basis + j * s;
    double acc = 0.0;
    for (size_t i = 0; i < s; ++i) acc += row[i] * x[i];
    out[j] = acc;
  }
}

/* DctPlan::inverse, transform.cpp:65-73: ascending j, zero coefficients skipped */
void dmo_dct_inverse(size_t s, const double* basis, const double* coeffs, double* out) {
  for (size_t i = 0; i < s; ++i) out[i] = 0.0;
  for (size_t j = 0; j < s; ++j) {
    const double c = coeffs[j];
    if (c == 0.0) continue;
    const double* row = basis + j * s;
    for (size_t i = 0; i < s; ++i) out[i] += c * row[i];
  }
}

typedef struct {
  double mag;
  uint32_t idx;
} mag_idx;

/* comparator of transform.cpp:128-133: larger |c| first, ties toward lower index */
static int cmp_mag_idx(const void* pa, const void* pb) {
  const mag_idx* a = (const mag_idx*)pa;
  const mag_idx* b = (const mag_idx*)pb;
  if (a->mag != b->mag) return a->mag > b->mag ? -1 : 1;
  return a->idx < b->idx ? -1 : (a->idx > b->idx ? 1 : 0);
}
static int cmp_u32(const void* pa, const void* pb) {
  const uint32_t a = *(const uint32_t*)pa, b = *(const uint32_t*)pb;
  return a < b ? -1 : (a > b ? 1 : 0);
}

/* extract_fast_components, transform.cpp:94-155 */
int dmo_extract_fast_components(const double* v, size_t len, size_t s, size_t top_k,
                                uint32_t* indices, double* coeffs, double* fast,
                                double* residual) {
  if (s == 0) return fail(DMO_CONFIG, "chunk size must be positive");
  if (top_k == 0 || top_k > s) {
    snprintf(g_err, sizeof g_err, "top_k %zu out of range for chunk size %zu", top_k, s);
    return DMO_CONFIG;
  }
  const size_t nc = dmo_num_chunks(len, s);
  double* basis = (double*)malloc(s * s * sizeof(double));
  double* row = (double*)malloc(s * sizeof(double));
  double* c = (double*)malloc(s * sizeof(double));
  double* sparse = (double*)malloc(s * sizeof(double));
  double* recon = (double*)malloc(s * sizeof(double));
  mag_idx* order = (mag_idx*)malloc(s * sizeof(mag_idx));
  uint32_t* sel = (uint32_t*)malloc(s * sizeof(uint32_t));
  dmo_dct_basis(s, basis);
  for (size_t ch = 0; ch < nc; ++ch) {
    /* chunk(): zero pad the tail, transform.cpp:27-32 */
    for (size_t i = 0; i < s; ++i) {
      const size_t g = ch * s + i;
      row[i] = g < len ? v[g] : 0.0;
    }
    dmo_dct_forward(s, basis, row, c);
    if (top_k == s) {
      /* full band: identity, exactly (transform.cpp:119-125) */
      for (size_t j = 0; j < s; ++j) {
        indices[ch * top_k + j] = (uint32_t)j;
        coeffs[ch * top_k + j] = c[j];
      }
      for (size_t i = 0; i < s; ++i) recon[i] = row[i];
    } else {
      for (size_t j = 0; j < s; ++j) {
        order[j].mag = fabs(c[j]);
        order[j].idx = (uint32_t)j;
      }
      qsort(order, s, sizeof(mag_idx), cmp_mag_idx);
      for (size_t q = 0; q < top_k; ++q) sel[q] = order[q].idx;
      qsort(sel, top_k, sizeof(uint32_t), cmp_u32);
      for (size_t j = 0; j < s; ++j) sparse[j] = 0.0;
      for (size_t q = 0; q < top_k; ++q) {
        const uint32_t j = sel[q];
        indices[ch * top_k + q] = j;
        coeffs[ch * top_k + q] = c[j];
        sparse[j] = c[j];
      }
      dmo_dct_inverse(s, basis, sparse, recon);
    }
    for (size_t i = 0; i < s; ++i) {
      const size_t g = ch * s + i;
      if (g < len) fast[g] = recon[i]; /* unchunk drops the pad */
    }
  }
  if (residual) {
    for (size_t i = 0; i < len; ++i) residual[i] = top_k == s ? 0.0 : v[i] - fast[i];
  }
  free(basis); free(row); free(c); free(sparse); free(recon); free(order); free(sel);
  return DMO_OK;
}

/* sign_transform, transform.cpp:157-161 */
void dmo_sign_transform(double* v, size_t n) {
  for (size_t i = 0; i < n; ++i) {
    const double x = v[i];
    v[i] = x > 0.0 ? 1.0 : (x < 0.0 ? -1.0 : 0.0);
  }
}

/* ======================= replicate.cpp ================================== */

/* replicate.cpp:35-42 */
size_t dmo_value_bits(int dtype) {
  switch (dtype) {
    case DMO_FP32: return 32;
    case DMO_FP16: return 16;
    case DMO_TERNARY: return 2;
  }
  return 32;
}

/* replicate.cpp:44-48 */
uint64_t dmo_wire_bytes(uint64_t n_values, uint64_t n_indices, int dtype) {
  const uint64_t bits = n_values * (uint64_t)dmo_value_bits(dtype) + n_indices * 32;
  return (bits + 7) / 8;
}

/* ReplicatorConfig::period, replicate.cpp:50-53 */
uint64_t dmo_period(double compression) {
  const long long p = llround(1.0 / compression);
  return p < 1 ? 1 : (uint64_t)p;
}

/* replicate.cpp:55-63 */
double dmo_narrow_to_fp32(double x) {
  if (isnan(x)) return x;
  const double kMax = 3.4028235677973366e38;
  if (fabs(x) >= kMax) return copysign(INFINITY, x);
  return (double)(float)x;
}

/* replicate.cpp:65-83 */
double dmo_narrow_to_fp16(double x) {
  if (isnan(x)) return x;
  const double a = fabs(x);
  if (a == 0.0) return x;
  const double sign = signbit(x) ? -1.0 : 1.0;
  if (a >= 65520.0) return sign * INFINITY;
  int e2;
  frexp(a, &e2);
  const int e = e2 - 1;
  const double ulp = ldexp(1.0, e >= -14 ? e - 10 : -24);
  const double q = a / ulp;
  const double r = nearbyint(q);
  const double res = r * ulp;
  if (res >= 65520.0) return sign * INFINITY;
  return sign * res;
}

/* replicate.cpp:87-102 */
uint16_t dmo_fp16_bits(double x) {
  const double v = dmo_narrow_to_fp16(x);
  const uint16_t sign = signbit(v) ? 0x8000 : 0;
  if (isnan(v)) return (uint16_t)(sign | 0x7e00);
  const double a = fabs(v);
  if (a == 0.0) return sign;
  if (isinf(v)) return (uint16_t)(sign | 0x7c00);
  if (a < 0x1.0p-14) {
    const uint16_t mant = (uint16_t)llround(ldexp(a, 24));
    return (uint16_t)(sign | mant);
  }
  const int e = ilogb(a);
  const double m = ldexp(a, -e);
  const uint16_t mant = (uint16_t)llround((m - 1.0) * 1024.0);
  return (uint16_t)(sign | ((e + 15) << 10) | mant);
}

/* condition_values, replicate.cpp:137-144 */
static void condition_values(double* values, uint64_t n, const dmo_rep_cfg* cfg) {
  if (cfg->sign_mode || cfg->transfer_dtype == DMO_TERNARY) dmo_sign_transform(values, n);
  if (cfg->transfer_dtype == DMO_FP16) {
    for (uint64_t i = 0; i < n; ++i) values[i] = dmo_narrow_to_fp16(values[i]);
  }
}

/* selection_count, replicate.cpp:146-156 */
static int64_t selection_count(double compression, uint64_t length) {
  const long long c = llround(compression * (double)length);
  if (c < 1) {
    snprintf(g_err, sizeof g_err,
             "compression %g selects no components from a vector of length %llu", compression,
             (unsigned long long)length);
    return -1;
  }
  return (uint64_t)c < length ? c : (int64_t)length;
}

int64_t dmo_value_count(const dmo_rep_cfg* cfg, uint64_t step, uint64_t len) {
  switch (cfg->scheme) {
    case DMO_FULL: return (int64_t)len;
    case DMO_DILOCO: return step % dmo_period(cfg->compression) != 0 ? 0 : (int64_t)len;
    case DMO_RANDOM: return selection_count(cfg->compression, len);
    case DMO_STRIDING: {
      const uint64_t n = dmo_period(cfg->compression);
      if (n > len) {
        snprintf(g_err, sizeof g_err, "stride period %llu exceeds vector length %llu",
                 (unsigned long long)n, (unsigned long long)len);
        return -1;
      }
      const uint64_t off = step % n;
      return off >= len ? 0 : (int64_t)((len - off + n - 1) / n);
    }
    case DMO_DEMO:
      if (cfg->chunk_size == 0) { fail(DMO_CONFIG, "chunk size must be positive"); return -1; }
      if (cfg->top_k == 0 || cfg->top_k > cfg->chunk_size) {
        snprintf(g_err, sizeof g_err, "top_k %llu out of range for chunk size %llu",
                 (unsigned long long)cfg->top_k, (unsigned long long)cfg->chunk_size);
        return -1;
      }
      return (int64_t)(dmo_num_chunks(len, cfg->chunk_size) * cfg->top_k);
  }
  fail(DMO_CONFIG, "unknown scheme");
  return -1;
}

/* selected_indices, replicate.cpp:160-185 */
int dmo_selected_indices(const dmo_rep_cfg* cfg, uint64_t step, uint32_t shard, uint64_t len,
                         uint32_t* out, uint64_t* count) {
  if (cfg->scheme == DMO_RANDOM) {
    const int64_t cnt = selection_count(cfg->compression, len);
    if (cnt < 0) return DMO_CONFIG;
    uint32_t* all = (uint32_t*)malloc((len ? len : 1) * sizeof(uint32_t));
    for (uint64_t i = 0; i < len; ++i) all[i] = (uint32_t)i;
    dmo_rng r;
    dmo_rng_init(&r, dmo_mix_seed3(cfg->seed, step, shard));
    /* Rng::shuffle, rng.hpp:40-45: full Fisher-Yates */
    for (uint64_t i = len; i > 1; --i) {
      const uint64_t j = dmo_rng_below(&r, i);
      const uint32_t t = all[i - 1];
      all[i - 1] = all[j];
      all[j] = t;
    }
    memcpy(out, all, (size_t)cnt * sizeof(uint32_t));
    free(all);
    qsort(out, (size_t)cnt, sizeof(uint32_t), cmp_u32);
    *count = (uint64_t)cnt;
    return DMO_OK;
  }
  if (cfg->scheme == DMO_STRIDING) {
    const uint64_t n = dmo_period(cfg->compression);
    if (n > len) {
      snprintf(g_err, sizeof g_err, "stride period %llu exceeds vector length %llu",
               (unsigned long long)n, (unsigned long long)len);
      return DMO_CONFIG;
    }
    const uint64_t off = step % n;
    uint64_t c = 0;
    for (uint64_t i = off; i < len; i += n) out[c++] = (uint32_t)i;
    *count = c;
    return DMO_OK;
  }
  return fail(DMO_CONFIG, "selected_indices applies to random and striding schemes only");
}

/* select_and_encode, replicate.cpp:187-237 */
int dmo_select_and_encode(const double* v, uint64_t len, const dmo_rep_cfg* cfg, uint64_t step,
                          uint32_t shard, uint32_t* freq_indices, double* values,
                          uint64_t* n_values, uint64_t* n_indices, uint64_t* bytes,
                          int32_t* empty, double* local_q) {
  *empty = 0;
  *n_indices = 0;
  *n_values = 0;
  switch (cfg->scheme) {
    case DMO_FULL:
      memcpy(values, v, len * sizeof(double));
      memcpy(local_q, v, len * sizeof(double));
      *n_values = len;
      break;
    case DMO_DILOCO:
      if (step % dmo_period(cfg->compression) != 0) {
        *empty = 1;
        for (uint64_t i = 0; i < len; ++i) local_q[i] = 0.0;
        break;
      }
      memcpy(values, v, len * sizeof(double));
      memcpy(local_q, v, len * sizeof(double));
      *n_values = len;
      break;
    case DMO_RANDOM:
    case DMO_STRIDING: {
      const int64_t cnt = dmo_value_count(cfg, step, len);
      if (cnt < 0) return DMO_CONFIG;
      uint32_t* idx = (uint32_t*)malloc(((size_t)cnt + 1) * sizeof(uint32_t));
      uint64_t c = 0;
      int rc = dmo_selected_indices(cfg, step, shard, len, idx, &c);
      if (rc) { free(idx); return rc; }
      for (uint64_t i = 0; i < len; ++i) local_q[i] = 0.0;
      for (uint64_t j = 0; j < c; ++j) {
        values[j] = v[idx[j]];
        local_q[idx[j]] = v[idx[j]];
      }
      *n_values = c;
      free(idx);
      break;
    }
    case DMO_DEMO: {
      int rc = dmo_extract_fast_components(v, len, cfg->chunk_size, cfg->top_k, freq_indices,
                                           values, local_q, NULL);
      if (rc) return rc;
      *n_values = dmo_num_chunks(len, cfg->chunk_size) * cfg->top_k;
      *n_indices = *n_values;
      break;
    }
    default:
      return fail(DMO_CONFIG, "unknown scheme");
  }
  condition_values(values, *n_values, cfg);
  *bytes = dmo_wire_bytes(*n_values, *n_indices, cfg->transfer_dtype);
  return DMO_OK;
}

/* decode_and_merge arithmetic, replicate.cpp:239-314 (metadata agreement checks
 * of :241-253 live with the caller, which holds the update headers) */
int dmo_decode_and_merge(const dmo_rep_cfg* cfg, uint64_t replicas, const double* const* values,
                         const uint32_t* const* freq_indices, uint64_t n_values, uint64_t len,
                         uint64_t step, uint32_t shard, double* q) {
  if (replicas == 0) return fail(DMO_PROTOCOL, "decode_and_merge needs at least one update");
  const double r = (double)replicas;
  for (uint64_t i = 0; i < len; ++i) q[i] = 0.0;
  switch (cfg->scheme) {
    case DMO_FULL:
    case DMO_DILOCO:
      if (n_values != len) return fail(DMO_PROTOCOL, "full update has the wrong length");
      for (uint64_t u = 0; u < replicas; ++u)
        for (uint64_t i = 0; i < len; ++i) q[i] += values[u][i];
      for (uint64_t i = 0; i < len; ++i) q[i] /= r;
      return DMO_OK;
    case DMO_RANDOM:
    case DMO_STRIDING: {
      const int64_t cnt = dmo_value_count(cfg, step, len);
      if (cnt < 0) return DMO_CONFIG;
      uint32_t* idx = (uint32_t*)malloc(((size_t)cnt + 1) * sizeof(uint32_t));
      uint64_t c = 0;
      int rc = dmo_selected_indices(cfg, step, shard, len, idx, &c);
      if (rc) { free(idx); return rc; }
      if (c != n_values) {
        free(idx);
        return fail(DMO_PROTOCOL, "selected value count does not match the derived index set");
      }
      for (uint64_t j = 0; j < c; ++j) {
        double acc = 0.0;
        for (uint64_t u = 0; u < replicas; ++u) acc += values[u][j];
        q[idx[j]] = acc / r;
      }
      free(idx);
      return DMO_OK;
    }
    case DMO_DEMO: {
      const uint64_t s = cfg->chunk_size, k = cfg->top_k;
      const uint64_t nc = dmo_num_chunks(len, s);
      if (n_values != nc * k)
        return fail(DMO_PROTOCOL, "frequency payload does not match the chunk layout");
      double* grid = (double*)calloc(nc * s + 1, sizeof(double));
      for (uint64_t u = 0; u < replicas; ++u) {
        for (uint64_t t = 0; t < n_values; ++t) {
          const uint64_t ch = t / k;
          const uint32_t j = freq_indices[u][t];
          if (j >= s) { free(grid); return fail(DMO_PROTOCOL, "frequency index out of range"); }
          grid[ch * s + j] += values[u][t];
        }
      }
      for (uint64_t i = 0; i < nc * s; ++i) grid[i] /= r;
      double* basis = (double*)malloc(s * s * sizeof(double));
      double* row = (double*)malloc(s * sizeof(double));
      dmo_dct_basis(s, basis);
      for (uint64_t ch = 0; ch < nc; ++ch) {
        dmo_dct_inverse(s, basis, grid + ch * s, row);
        for (uint64_t i = 0; i < s; ++i)
          if (ch * s + i < len) q[ch * s + i] = row[i];
      }
      free(basis); free(row); free(grid);
      return DMO_OK;
    }
  }
  return fail(DMO_CONFIG, "unknown scheme");
}

static void put_u32(uint8_t* o, uint32_t v) { for (int i = 0; i < 4; ++i) o[i] = (uint8_t)(v >> (8 * i)); }

/* serialize, replicate.cpp:316-356; returns total bytes (9 + body) */
uint64_t dmo_serialize(int scheme, const uint32_t* freq_indices, uint64_t n_indices,
                       const double* values, uint64_t n_values, int dtype, uint8_t* out) {
  uint64_t off = 0;
  out[off++] = (uint8_t)scheme;
  for (int i = 0; i < 8; ++i) out[off++] = (uint8_t)(n_values >> (8 * i));
  if (scheme == DMO_DEMO) {
    for (uint64_t i = 0; i < n_indices; ++i, off += 4) put_u32(out + off, freq_indices[i]);
  }
  if (dtype == DMO_FP32) {
    for (uint64_t i = 0; i < n_values; ++i, off += 4) {
      float f = (float)dmo_narrow_to_fp32(values[i]);
      uint32_t b;
      memcpy(&b, &f, 4);
      put_u32(out + off, b);
    }
  } else if (dtype == DMO_FP16) {
    for (uint64_t i = 0; i < n_values; ++i) {
      const uint16_t b = dmo_fp16_bits(values[i]);
      out[off++] = (uint8_t)(b & 0xff);
      out[off++] = (uint8_t)(b >> 8);
    }
  } else {
    uint8_t pack = 0;
    int filled = 0;
    for (uint64_t i = 0; i < n_values; ++i) {
      const double v = values[i];
      const uint8_t code = v > 0.0 ? 1 : (v < 0.0 ? 2 : 0);
      pack |= (uint8_t)(code << (2 * filled));
      if (++filled == 4) { out[off++] = pack; pack = 0; filled = 0; }
    }
    if (filled) out[off++] = pack;
  }
  return off;
}

/* ======================= vec.cpp / optim.cpp ============================ */

/* require_finite, vec.cpp:7-16: first offending index or -1 */
int64_t dmo_first_nonfinite(const double* v, uint64_t n) {
  for (uint64_t i = 0; i < n; ++i)
    if (!isfinite(v[i])) return (int64_t)i;
  return -1;
}

/* demo_sgd_prepare, optim.cpp:18-43 */
int dmo_demo_sgd_prepare(double* m, const double* grad, uint64_t len, double beta,
                         const dmo_rep_cfg* cfg, uint64_t step, uint32_t shard,
                         uint32_t* freq_indices, double* values, uint64_t* n_values,
                         uint64_t* bytes, int32_t* empty, double* local_q,
                         double* m_accum_trace, int64_t* bad_index) {
  const int64_t bad = dmo_first_nonfinite(grad, len);
  if (bad_index) *bad_index = bad;
  if (bad >= 0) {
    snprintf(g_err, sizeof g_err, "gradient contains a non-finite value (%g at index %lld)",
             grad[bad], (long long)bad);
    return DMO_TRAINING;
  }
  for (uint64_t i = 0; i < len; ++i) m[i] = beta * m[i] + grad[i];
  if (m_accum_trace) memcpy(m_accum_trace, m, len * sizeof(double));
  uint64_t n_idx = 0;
  int rc = dmo_select_and_encode(m, len, cfg, step, shard, freq_indices, values, n_values,
                                 &n_idx, bytes, empty, local_q);
  if (rc) return rc;
  for (uint64_t i = 0; i < len; ++i) m[i] -= local_q[i];
  return DMO_OK;
}

/* demo_sgd_apply, optim.cpp:45-49 */
void dmo_demo_sgd_apply(double* params, const double* q, uint64_t n, double lr) {
  for (uint64_t i = 0; i < n; ++i) params[i] -= lr * q[i];
}

/* adamw_apply, optim.cpp:57-74 */
void dmo_adamw_apply(double* params, double* exp_avg, double* exp_avg_sq, uint64_t* steps,
                     const double* grad, const double* local_q, const double* merged,
                     uint64_t n, double beta1, double beta2, double eps, double weight_decay,
                     double lr) {
  *steps += 1;
  const double bc1 = 1.0 - pow(beta1, (double)*steps);
  const double bc2 = 1.0 - pow(beta2, (double)*steps);
  for (uint64_t i = 0; i < n; ++i) {
    const double g = merged != NULL ? grad[i] - local_q[i] + merged[i] : grad[i];
    exp_avg[i] = beta1 * exp_avg[i] + (1.0 - beta1) * g;
    exp_avg_sq[i] = beta2 * exp_avg_sq[i] + (1.0 - beta2) * g * g;
    const double m_hat = exp_avg[i] / bc1;
    const double v_hat = exp_avg_sq[i] / bc2;
    params[i] -= lr * (m_hat / (sqrt(v_hat) + eps));
    if (weight_decay != 0.0) params[i] -= lr * weight_decay * params[i];
  }
}

/* baseline_sgd_step, optim.cpp:76-86 */
int dmo_baseline_sgd_step(double* params, double* m, const double* grad, uint64_t n,
                          double beta, double lr) {
  if (dmo_first_nonfinite(grad, n) >= 0) return fail(DMO_TRAINING, "gradient is not finite");
  for (uint64_t i = 0; i < n; ++i) {
    const double v = beta * m[i] + grad[i];
    params[i] -= lr * v;
    m[i] = 0.0;
  }
  return DMO_OK;
}

/* baseline_adamw_step, optim.cpp:88-93 */
int dmo_baseline_adamw_step(double* params, double* exp_avg, double* exp_avg_sq, uint64_t* steps,
                            const double* grad, uint64_t n, double beta1, double beta2,
                            double eps, double weight_decay, double lr) {
  if (dmo_first_nonfinite(grad, n) >= 0) return fail(DMO_TRAINING, "gradient is not finite");
  dmo_adamw_apply(params, exp_avg, exp_avg_sq, steps, grad, grad, NULL, n, beta1, beta2, eps,
                  weight_decay, lr);
  return DMO_OK;
}

/* grad_reduce_scatter, cluster.cpp:63-91 with mean_of, vec.cpp:18-26 */
int dmo_grad_reduce_scatter(uint64_t members, uint64_t len, const double* const* grads,
                            double* shards) {
  if (members == 0) return fail(DMO_PROTOCOL, "reduce-scatter over an empty group");
  if (len % members != 0) return fail(DMO_PROTOCOL, "vector length is not divisible into shards");
  const double n = (double)members;
  for (uint64_t i = 0; i < len; ++i) {
    double acc = 0.0;
    for (uint64_t a = 0; a < members; ++a) acc += grads[a][i];
    shards[i] = acc / n; /* shards laid out member-major == the padded vector order */
  }
  return DMO_OK;
}
