// inst_u32.cu -- explicit instantiation of the SquareSort engine for uint32_t keys (compiled
// as its own translation unit so the library builds in parallel).
#include "engine.cuh"

namespace sq {
template void sort_device<uint32_t, false>(uint32_t*, uint32_t*, size_t, uint64_t, cudaStream_t);

void debug_level_u32(const uint32_t* src, uint32_t* dst, size_t n, uint64_t seed, uint32_t* pivots_out,
                     uint32_t* bucend_out, uint32_t* info_out, cudaStream_t st) {
  Arena ar(st);
  uint32_t* work = (uint32_t*)ar.alloc(n * 4);
  SQ_CUDA(cudaMemcpyAsync(work, src, n * 4, cudaMemcpyDeviceToDevice, st));
  Engine<uint32_t, false> eng(st, ar, work, nullptr, n);
  DebugOut dbg{dst, pivots_out, bucend_out, info_out};
  std::vector<Seg> top = {{0, (uint32_t)n, root_key(seed)}};
  eng.run_level(top, 0, 0, &dbg);
  SQ_CUDA(cudaStreamSynchronize(st));
}
}  // namespace sq
