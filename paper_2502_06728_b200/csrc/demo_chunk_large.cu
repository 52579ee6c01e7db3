// demo_chunk_large.cu -- instantiations for chunk sizes 64 < s <= 256 (E = 4, 8; CH = 1).
// Not on any configured hot path (the configs use s = 64); present so every chunk size
// the reference accepts runs on the device.
#include "demo_chunk.cuh"

namespace dmb {
namespace {
using chunk_impl::launch_t;

template <ChunkMode MODE>
void dispatch_large(const ChunkArgs& a, cudaStream_t stream) {
  const int s = a.geo.s;
  if (s <= 128) launch_t<4, 1, MODE>(a, stream);
  else launch_t<8, 1, MODE>(a, stream);
}
}  // namespace

void launch_chunk_large(ChunkMode mode, const ChunkArgs& a, cudaStream_t stream) {
  switch (mode) {
    case ChunkMode::EncodeSgd: dispatch_large<ChunkMode::EncodeSgd>(a, stream); break;
    case ChunkMode::EncodeAdam: dispatch_large<ChunkMode::EncodeAdam>(a, stream); break;
    case ChunkMode::StepSgd: dispatch_large<ChunkMode::StepSgd>(a, stream); break;
    case ChunkMode::StepAdam: dispatch_large<ChunkMode::StepAdam>(a, stream); break;
    case ChunkMode::MergeSgd: dispatch_large<ChunkMode::MergeSgd>(a, stream); break;
    case ChunkMode::MergeAdam: dispatch_large<ChunkMode::MergeAdam>(a, stream); break;
  }
}
}  // namespace dmb
