// inst_u64.cu -- explicit instantiation of the SquareSort engine for uint64_t keys (its own
// translation unit, so the library builds in parallel).
#include "engine.cuh"

namespace sq {
template void sort_engine<uint64_t, false, false>(uint64_t*, uint32_t*, size_t, uint64_t, cudaStream_t);
template void debug_level_engine<uint64_t, false>(const uint64_t*, uint64_t*, size_t, uint64_t, uint64_t*, uint32_t*,
                                                  uint32_t*, cudaStream_t);
}  // namespace sq
