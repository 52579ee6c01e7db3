// demo_chunk_small.cu -- instantiations for chunk sizes s <= 64 (E = 1, 2; CH = 4)
// and the mode dispatcher.
#include <cstdlib>

#include "demo_chunk.cuh"

namespace dmb {
// DMB_TC=0 forces the SIMT path (A/B checks); read per launch so tests can flip it
bool tc_enabled() {
  const char* e = std::getenv("DMB_TC");
  return !(e && e[0] == '0');
}

// DMB_FORCE_FP64=1 (tests): every chunk takes the exact FP64 re-derivation path
static bool force_fp64_env() {
  const char* e = std::getenv("DMB_FORCE_FP64");
  return e && e[0] == '1';
}

void launch_chunk_kernel(ChunkMode mode, const ChunkArgs& a_in, cudaStream_t stream) {
  ChunkArgs a = a_in;
  if (force_fp64_env()) a.force_fp64 = 1;
  if (a.n_src > 0) {
    // the shard group's reduce-scatter fused into the gradient load: the tensor-core kernel
    // averages the members' tiles and writes the mean to a.g; the partial last chunk's mean
    // comes first (its SIMT pass reads a.g).  Anywhere else the mean is a pass of its own.
    const bool fused = tc_enabled() && a.fb_list && a.fb_count && tc3_supported(mode, a);
    const uint64_t from = fused ? (a.geo.len / a.geo.s) * a.geo.s : 0;
    if (from < a.geo.len) {
      const float* tails[kMaxGradSrc];
      for (int q = 0; q < a.n_src; ++q) tails[q] = a.g_src[q] + from;
      launch_grad_mean(tails, a.n_src, a.geo.len - from, const_cast<float*>(a.g) + from, stream);
    }
    if (!fused) a.n_src = 0;
  }
  if (tc_enabled() && a.fb_list && a.fb_count && tc3_supported(mode, a)) {
    // warp-specialised tensor-core kernel; the chunks its FP32 bound cannot certify are
    // re-derived exactly by the FP64 fix-up kernel; a partial last chunk (its own
    // length and basis) goes through the SIMT kernel
    // a merge never defers: it leaves the fix-up list to an encode that may be running
    // concurrently on another stream
    if (mode != ChunkMode::MergeAdam && mode != ChunkMode::MergeSgd) cudaMemsetAsync(a.fb_count, 0, sizeof(unsigned), stream);
    timer_begin(stream);
    launch_tc3_kernel(mode, a, stream);
    timer_end(stream);
    launch_fix64_kernel(mode, a, stream);
    if (a.geo.len % a.geo.s) {
      ChunkArgs tail = a;
      tail.first_chunk = a.geo.nchunks - 1;
      launch_chunk_simt(mode, tail, stream);
    }
    return;
  }
  if (tc_enabled() && a.fb_list && a.fb_count && tc_supported(mode, a)) {
    cudaMemsetAsync(a.fb_count, 0, sizeof(unsigned), stream);
    timer_begin(stream);
    launch_tc_kernel(mode, a, stream);
    timer_end(stream);
    ChunkArgs fix = a;
    fix.list = a.fb_list;
    fix.list_count = a.fb_count;
    // the SIMT kernel certifies its own FP32 coefficients (a tighter bound than the
    // tensor-core one) and re-derives in FP64 only what that bound cannot settle
    fix.force_fp64 = a.force_fp64;
    launch_chunk_simt(mode, fix, stream);
    return;
  }
  launch_chunk_simt(mode, a, stream);
}

void launch_chunk_large(ChunkMode mode, const ChunkArgs& a, cudaStream_t stream);
namespace {
using chunk_impl::launch_t;

template <ChunkMode MODE>
void dispatch_small(const ChunkArgs& a, cudaStream_t stream) {
  if (a.geo.s <= 32) launch_t<1, 4, MODE>(a, stream);
  else launch_t<2, 4, MODE>(a, stream);
}
}  // namespace

template <ChunkMode MODE>
void dispatch_list(const ChunkArgs& a, cudaStream_t stream) {
  launch_t<2, 1, MODE>(a, stream);
}

void launch_chunk_simt(ChunkMode mode, const ChunkArgs& a, cudaStream_t stream) {
  if (a.list) {  // FP64 re-derivation of the chunks the tensor-core kernel could not certify
    switch (mode) {
      case ChunkMode::EncodeSgd: dispatch_list<ChunkMode::EncodeSgd>(a, stream); break;
      case ChunkMode::EncodeAdam: dispatch_list<ChunkMode::EncodeAdam>(a, stream); break;
      case ChunkMode::StepSgd: dispatch_list<ChunkMode::StepSgd>(a, stream); break;
      case ChunkMode::StepAdam: dispatch_list<ChunkMode::StepAdam>(a, stream); break;
      case ChunkMode::MergeSgd: dispatch_list<ChunkMode::MergeSgd>(a, stream); break;
      case ChunkMode::MergeAdam: dispatch_list<ChunkMode::MergeAdam>(a, stream); break;
    }
    return;
  }
  if (a.geo.s > 64) {
    launch_chunk_large(mode, a, stream);
    return;
  }
  switch (mode) {
    case ChunkMode::EncodeSgd: dispatch_small<ChunkMode::EncodeSgd>(a, stream); break;
    case ChunkMode::EncodeAdam: dispatch_small<ChunkMode::EncodeAdam>(a, stream); break;
    case ChunkMode::StepSgd: dispatch_small<ChunkMode::StepSgd>(a, stream); break;
    case ChunkMode::StepAdam: dispatch_small<ChunkMode::StepAdam>(a, stream); break;
    case ChunkMode::MergeSgd: dispatch_small<ChunkMode::MergeSgd>(a, stream); break;
    case ChunkMode::MergeAdam: dispatch_small<ChunkMode::MergeAdam>(a, stream); break;
  }
}
}  // namespace dmb
