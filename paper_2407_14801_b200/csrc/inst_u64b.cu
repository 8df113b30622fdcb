// inst_u64b.cu -- explicit instantiation of the SquareSort engine for uint64_t keys with the counting-sort base case (its own
// translation unit, so the library builds in parallel).
#include "engine.cuh"

namespace sq {
template void sort_engine<uint64_t, false, true>(uint64_t*, uint32_t*, size_t, uint64_t, cudaStream_t);
}  // namespace sq
