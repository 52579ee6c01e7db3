// toy_models.cu -- the reference's gradient producers (model.hpp / model.cpp) on the device, for
// the trainer loop (paper_2502_06728_b200/trainer.py, trainer.cpp:49-90):
//
//   quadratic  loss = mean_i 0.5 ||theta - x_i||^2, grad = theta - mean(x)  (model.cpp:107-119, :152-161)
//   mlp        fully connected, tanh / relu hidden, linear output, MSE or softmax cross entropy,
//              parameters W0 b0 W1 b1 ... with W row major (out x in)      (model.cpp:42-105, :163-203)
//
// One CTA per worker, every worker of the emulated cluster in ONE launch: worker w evaluates at
// the parameter row w / workers_per_row (its node's parameters) on the mini batch BatchStream
// assigns to (step, rank w) (dataset.cpp:141-151), read straight from the device-resident pool
// through the device copy of the permutation -- no host work per step.  The arithmetic is FP64
// in the reference's operation order (no contraction: __dadd_rn / __dmul_rn): every forward
// dot product is one thread's ascending sum, every gradient element is owned by one thread that
// accumulates the examples in batch order, the per-example losses are summed in order by one
// thread.  The only differences from the reference's FP64 evaluation are the device's tanh / exp
// / log (within an ulp of libm) and the FP32 storage of the parameters and of the returned
// gradient.
#include "dmb_internal.cuh"

namespace dmb {
namespace {

constexpr int kToyThreads = 256;

__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }

__device__ __forceinline__ uint64_t example_of(const int64_t* order, uint64_t order_len, uint64_t base,
                                               uint64_t j) {
  return order ? (uint64_t)order[(base + j) % order_len] : j;  // dataset.cpp:145-149
}

// quadratic: thread d owns coordinate d (mean over the batch in order); loss per example by one
// thread each (ascending d), summed in batch order by thread 0
__global__ void __launch_bounds__(kToyThreads) quadratic_kernel(ToyArgs a) {
  extern __shared__ double sq[];  // batch entries
  const uint64_t w = blockIdx.x;
  const float* theta = a.params + (w / a.workers_per_row) * a.params_stride;
  const uint32_t D = a.dims[0];
  const uint64_t base = (a.step * a.world + w) * a.batch;
  const double* X = a.inputs;
  for (uint64_t i = threadIdx.x; i < a.batch; i += blockDim.x) {
    const double* x = X + example_of(a.order, a.order_len, base, i) * D;
    double s = 0.0;
    for (uint32_t d = 0; d < D; ++d) {
      const double diff = (double)theta[d] - x[d];
      s = dadd(s, dmul(diff, diff));
    }
    sq[i] = s;
  }
  if (a.grad) {
    float* g = a.grad + w * a.grad_stride;
    for (uint64_t d = threadIdx.x; d < a.grad_len; d += blockDim.x) {
      if (d >= D) {
        g[d] = 0.0f;  // the padding receives exact zeros (model.hpp:56-57)
        continue;
      }
      double sum = 0.0;
      for (uint64_t i = 0; i < a.batch; ++i) sum = dadd(sum, X[example_of(a.order, a.order_len, base, i) * D + d]);
      g[d] = (float)((double)theta[d] - sum / (double)a.batch);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double acc = 0.0;
    for (uint64_t i = 0; i < a.batch; ++i) acc = dadd(acc, dmul(0.5, sq[i]));
    a.loss[w] = acc / (double)a.batch;
  }
}

__device__ __forceinline__ double activate(int act, double z) { return act == 0 ? tanh(z) : (z > 0.0 ? z : 0.0); }
__device__ __forceinline__ double activate_grad(int act, double y) {
  return act == 0 ? 1.0 - dmul(y, y) : (y > 0.0 ? 1.0 : 0.0);
}

// mlp: per example, layer by layer in shared memory; the gradient accumulates in shared memory
// (FP64, one owner thread per element) and is rounded to FP32 once at the end.
// shared layout: gacc[P] | acts[sum dims] | delta[maxd] | delta2[maxd] | probs[out] | lsum
__global__ void __launch_bounds__(kToyThreads) mlp_kernel(ToyArgs a) {
  extern __shared__ double sm[];
  const uint64_t w = blockIdx.x;
  const float* P = a.params + (w / a.workers_per_row) * a.params_stride;
  const int L = (int)a.n_dims - 1;  // layers
  uint32_t act_off[kToyMaxDims];
  uint64_t par_off[kToyMaxDims];
  uint32_t tot = 0, maxd = 0;
  uint64_t pc = 0;
  for (int l = 0; l <= L; ++l) {
    act_off[l] = tot;
    tot += a.dims[l];
    maxd = a.dims[l] > maxd ? a.dims[l] : maxd;
    par_off[l] = pc;
    if (l < L) pc += (uint64_t)a.dims[l + 1] * a.dims[l] + a.dims[l + 1];
  }
  const bool want_grad = a.grad != nullptr;
  double* gacc = sm;
  double* acts = gacc + (want_grad ? pc : 0);
  double* delta = acts + tot;
  double* delta2 = delta + maxd;
  double* probs = delta2 + maxd;
  const uint32_t out_dim = a.dims[L];
  if (want_grad)
    for (uint64_t e = threadIdx.x; e < pc; e += blockDim.x) gacc[e] = 0.0;
  const uint64_t base = (a.step * a.world + w) * a.batch;
  const double inv_b = 1.0 / (double)a.batch;
  double loss_acc = 0.0;  // thread 0
  for (uint64_t i = 0; i < a.batch; ++i) {
    const uint64_t ex = example_of(a.order, a.order_len, base, i);
    const double* x = a.inputs + ex * a.dims[0];
    for (uint32_t c = threadIdx.x; c < a.dims[0]; c += blockDim.x) acts[c] = x[c];
    __syncthreads();
    for (int l = 0; l < L; ++l) {  // model.cpp:53-73
      const uint32_t in = a.dims[l], out = a.dims[l + 1];
      const float* W = P + par_off[l];
      const float* b = W + (uint64_t)out * in;
      const double* al = acts + act_off[l];
      double* an = acts + act_off[l + 1];
      const bool hidden = l + 1 < L;
      for (uint32_t r = threadIdx.x; r < out; r += blockDim.x) {
        double z = (double)b[r];
        const float* row = W + (uint64_t)r * in;
        for (uint32_t c = 0; c < in; ++c) z = dadd(z, dmul((double)row[c], al[c]));
        an[r] = hidden ? activate(a.activation, z) : z;
      }
      __syncthreads();
    }
    const double* o = acts + act_off[L];
    if (threadIdx.x == 0) {  // example_loss, model.cpp:75-105
      double li;
      if (a.loss_kind == 1) {
        double m = o[0];
        for (uint32_t r = 1; r < out_dim; ++r) m = o[r] > m ? o[r] : m;
        double denom = 0.0;
        for (uint32_t r = 0; r < out_dim; ++r) {
          probs[r] = exp(o[r] - m);
          denom = dadd(denom, probs[r]);
        }
        for (uint32_t r = 0; r < out_dim; ++r) probs[r] = probs[r] / denom;
        li = -log(probs[a.labels[ex]]);
      } else {
        const double* t = a.targets + ex * out_dim;
        double acc = 0.0;
        for (uint32_t r = 0; r < out_dim; ++r) {
          const double d = o[r] - t[r];
          acc = dadd(acc, dmul(d, d));
        }
        li = dmul(0.5, acc);
      }
      loss_acc = dadd(loss_acc, li);
    }
    if (!want_grad) {
      __syncthreads();
      continue;
    }
    __syncthreads();
    for (uint32_t r = threadIdx.x; r < out_dim; r += blockDim.x) {  // model.cpp:170-180
      if (a.loss_kind == 1)
        delta[r] = dmul(probs[r] - ((uint32_t)a.labels[ex] == r ? 1.0 : 0.0), inv_b);
      else
        delta[r] = dmul(o[r] - a.targets[ex * out_dim + r], inv_b);
    }
    __syncthreads();
    double* dcur = delta;
    double* dprev = delta2;
    for (int l = L - 1; l >= 0; --l) {  // model.cpp:183-199
      const uint32_t in = a.dims[l], out = a.dims[l + 1];
      const double* al = acts + act_off[l];
      double* gW = gacc + par_off[l];
      double* gb = gW + (uint64_t)out * in;
      const uint64_t nw = (uint64_t)out * in;
      for (uint64_t e = threadIdx.x; e < nw + out; e += blockDim.x) {
        if (e < nw) {
          const uint64_t r = e / in, c = e - r * in;
          gW[e] = dadd(gW[e], dmul(dcur[r], al[c]));
        } else {
          gb[e - nw] = dadd(gb[e - nw], dcur[e - nw]);
        }
      }
      if (l == 0) break;
      const float* W = P + par_off[l];
      for (uint32_t c = threadIdx.x; c < in; c += blockDim.x) {
        double s = 0.0;
        for (uint32_t r = 0; r < out; ++r) s = dadd(s, dmul((double)W[(uint64_t)r * in + c], dcur[r]));
        dprev[c] = dmul(s, activate_grad(a.activation, al[c]));
      }
      __syncthreads();
      double* t = dcur;
      dcur = dprev;
      dprev = t;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) a.loss[w] = loss_acc / (double)a.batch;
  if (want_grad) {
    float* g = a.grad + w * a.grad_stride;
    for (uint64_t e = threadIdx.x; e < a.grad_len; e += blockDim.x) g[e] = e < pc ? (float)gacc[e] : 0.0f;
  }
}

}  // namespace

uint64_t toy_smem_bytes(const ToyArgs& a) {
  if (a.kind == 0) return a.batch * 8;
  uint64_t tot = 0, maxd = 0, pc = 0;
  for (uint32_t l = 0; l < a.n_dims; ++l) {
    tot += a.dims[l];
    maxd = a.dims[l] > maxd ? a.dims[l] : maxd;
    if (l + 1 < a.n_dims) pc += (uint64_t)a.dims[l + 1] * a.dims[l] + a.dims[l + 1];
  }
  return 8 * ((a.grad ? pc : 0) + tot + 2 * maxd + a.dims[a.n_dims - 1]);
}

int launch_toy(const ToyArgs& a, cudaStream_t stream) {
  const uint64_t smem = toy_smem_bytes(a);
  if (a.kind == 0) {
    if (smem > 48 * 1024) cudaFuncSetAttribute(quadratic_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    quadratic_kernel<<<(unsigned)a.workers, kToyThreads, smem, stream>>>(a);
  } else {
    if (smem > 48 * 1024) cudaFuncSetAttribute(mlp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    mlp_kernel<<<(unsigned)a.workers, kToyThreads, smem, stream>>>(a);
  }
  count_launches(1);
  return 0;
}

}  // namespace dmb
