// inst_pairsb.cu -- explicit instantiation of the SquareSort engine for uint32_t keys with uint32_t values with the counting-sort base case (its own
// translation unit, so the library builds in parallel).
#include "engine.cuh"

namespace sq {
template void sort_engine<uint32_t, true, true>(uint32_t*, uint32_t*, size_t, uint64_t, cudaStream_t);
}  // namespace sq
