// transform.cu -- the transform.hpp:13-74 surface of the reference on the device (FP32 vectors):
// chunk / unchunk (transform.cpp:17-39), the orthonormal DCT-II and its inverse on batches of
// vectors (DctPlan::forward / inverse, transform.cpp:41-80), sign_transform (:157-161) and the
// residual of extract_fast_components (:147-153).  The DCTs accumulate in FP64 in the
// reference's operation order (forward: acc = 0, acc + B[j][i] x[i] for ascending i; inverse:
// ascending j, zero coefficients skipped) from the host's libm basis, so on the same inputs
// they are bit-exact with the reference before the final rounding to FP32.
#include "dmb_internal.cuh"

namespace dmb {
namespace {

constexpr int kT = 256;

__global__ void chunk_kernel(const float* __restrict__ v, uint64_t len, uint64_t padded, float* __restrict__ rows) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < padded; i += stride)
    rows[i] = i < len ? v[i] : 0.0f;
}

__global__ void copy_kernel(const float* __restrict__ a, uint64_t n, float* __restrict__ out) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) out[i] = a[i];
}

// one CTA per vector: x (FP64 in shared memory) -> out[j] = sum_i B[j][i] x[i], ascending i
__global__ void __launch_bounds__(kT) dct2_kernel(const float* __restrict__ x, uint64_t n,
                                                  const double* __restrict__ BT, float* __restrict__ out) {
  extern __shared__ double xs[];
  const float* xv = x + blockIdx.x * n;
  for (uint64_t i = threadIdx.x; i < n; i += kT) xs[i] = (double)xv[i];
  __syncthreads();
  for (uint64_t j = threadIdx.x; j < n; j += kT) {
    double acc = 0.0;
    for (uint64_t i = 0; i < n; ++i) acc = __dadd_rn(acc, __dmul_rn(BT[i * n + j], xs[i]));  // B[j][i]
    out[blockIdx.x * n + j] = (float)acc;
  }
}

// one CTA per vector: out[i] = sum over j with c_j != 0 of c_j B[j][i], ascending j
__global__ void __launch_bounds__(kT) idct3_kernel(const float* __restrict__ c, uint64_t n,
                                                   const double* __restrict__ B, float* __restrict__ out) {
  extern __shared__ double cs[];
  const float* cv = c + blockIdx.x * n;
  for (uint64_t j = threadIdx.x; j < n; j += kT) cs[j] = (double)cv[j];
  __syncthreads();
  for (uint64_t i = threadIdx.x; i < n; i += kT) {
    double acc = 0.0;
    for (uint64_t j = 0; j < n; ++j) {
      const double cj = cs[j];
      if (cj == 0.0) continue;  // transform.cpp:69 (uniform across the CTA)
      acc = __dadd_rn(acc, __dmul_rn(cj, B[j * n + i]));
    }
    out[blockIdx.x * n + i] = (float)acc;
  }
}

__global__ void sign_kernel(float* __restrict__ v, uint64_t n) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) v[i] = sign_of(v[i]);
}

__global__ void residual_kernel(const float* __restrict__ v, const float* __restrict__ fast, uint64_t n,
                                bool full_band, float* __restrict__ res) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    res[i] = full_band ? 0.0f : v[i] - fast[i];
}

unsigned grid_of(uint64_t n) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const uint64_t want = (n + kT - 1) / kT, cap = (uint64_t)sms * 8;
  return (unsigned)(want < cap ? (want ? want : 1) : cap);
}

}  // namespace

void launch_chunk(const float* v, uint64_t len, uint64_t padded, float* rows, cudaStream_t st) {
  count_launches(1);
  chunk_kernel<<<grid_of(padded), kT, 0, st>>>(v, len, padded, rows);
}
void launch_copy(const float* a, uint64_t n, float* out, cudaStream_t st) {
  count_launches(1);
  copy_kernel<<<grid_of(n), kT, 0, st>>>(a, n, out);
}
void launch_dct(bool inverse, const float* in, uint64_t n, uint64_t count, const Basis& b, float* out,
                cudaStream_t st) {
  count_launches(1);
  const size_t smem = n * sizeof(double);
  if (inverse) idct3_kernel<<<(unsigned)count, kT, smem, st>>>(in, n, b.B64, out);
  else dct2_kernel<<<(unsigned)count, kT, smem, st>>>(in, n, b.B64T, out);
}
void launch_sign(float* v, uint64_t n, cudaStream_t st) {
  count_launches(1);
  sign_kernel<<<grid_of(n), kT, 0, st>>>(v, n);
}
void launch_residual(const float* v, const float* fast, uint64_t n, bool full_band, float* res, cudaStream_t st) {
  count_launches(1);
  residual_kernel<<<grid_of(n), kT, 0, st>>>(v, fast, n, full_band, res);
}

}  // namespace dmb
