// inst_pairs.cu -- explicit instantiation of the SquareSort engine for uint32_t keys with uint32_t values (its own
// translation unit, so the library builds in parallel).
#include "engine.cuh"

namespace sq {
template void sort_engine<uint32_t, true, false>(uint32_t*, uint32_t*, size_t, uint64_t, cudaStream_t);
}  // namespace sq
