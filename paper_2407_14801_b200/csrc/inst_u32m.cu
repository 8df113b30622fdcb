// inst_u32m.cu -- explicit instantiation of the SquareSort engine for uint32_t keys with the merge-sort base case (its own
// translation unit, so the library builds in parallel).
#include "engine.cuh"

namespace sq {
template void sort_engine<uint32_t, false, false>(uint32_t*, uint32_t*, size_t, uint64_t, cudaStream_t);
template void debug_level_engine<uint32_t, false>(const uint32_t*, uint32_t*, size_t, uint64_t, uint32_t*, uint32_t*,
                                                  uint32_t*, cudaStream_t);
}  // namespace sq
