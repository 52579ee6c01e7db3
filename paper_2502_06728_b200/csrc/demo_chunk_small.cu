// demo_chunk_small.cu -- instantiations for chunk sizes s <= 64 (E = 1, 2; CH = 4)
// and the mode dispatcher.
#include "demo_chunk.cuh"

namespace dmb {
void launch_chunk_large(ChunkMode mode, const ChunkArgs& a, cudaStream_t stream);
namespace {
using chunk_impl::launch_t;

template <ChunkMode MODE>
void dispatch_small(const ChunkArgs& a, cudaStream_t stream) {
  if (a.geo.s <= 32) launch_t<1, 4, MODE>(a, stream);
  else launch_t<2, 4, MODE>(a, stream);
}
}  // namespace

void launch_chunk_kernel(ChunkMode mode, const ChunkArgs& a, cudaStream_t stream) {
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
