// Shared-memory scatter/atomic microbenchmarks on B200 (sm_100a): cycles per
// warp instruction per SM for the primitives a counting-sort base case would
// be made of (random STS, shared atomics with and without return, match.any
// on wide values).  Not part of the product; informs DESIGN.md section 8.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define ITERS 1024
#define UNROLL 8
constexpr int TBL = 8192;

__device__ __forceinline__ uint32_t hsh(uint32_t x) { return x * 2654435761u; }

template <int OP>
__global__ void k(uint32_t* out, uint32_t seed) {
  extern __shared__ uint32_t s[];
  const int t = threadIdx.x;
  for (int i = t; i < TBL * 2; i += blockDim.x) s[i] = i;
  __syncthreads();
  uint32_t a = hsh(seed ^ t), b = hsh(a + 1), c = hsh(b + 1), d = hsh(c + 1);
  uint32_t acc = 0;
  long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int u = 0; u < UNROLL; u++) {
      // four independent random streams per thread
      a = a * 1664525u + 1013904223u; b = b * 1664525u + 1013904223u;
      c = c * 1664525u + 1013904223u; d = d * 1664525u + 1013904223u;
      const uint32_t ia = a >> 19, ib = b >> 19, ic = c >> 19, id = d >> 19;  // 13 bits
      if (OP == 0) {  // ATOMS.ADD with return, random over 8K words
        acc += atomicAdd(&s[ia], 1u); acc += atomicAdd(&s[ib], 1u);
        acc += atomicAdd(&s[ic], 1u); acc += atomicAdd(&s[id], 1u);
      } else if (OP == 1) {  // RED (no return)
        atomicAdd(&s[ia], 1u); atomicAdd(&s[ib], 1u); atomicAdd(&s[ic], 1u); atomicAdd(&s[id], 1u);
      } else if (OP == 2) {  // STS random
        s[ia] = a; s[ib] = b; s[ic] = c; s[id] = d;
      } else if (OP == 3) {  // LDS random (independent)
        acc += s[ia] ^ s[ib] ^ s[ic] ^ s[id];
      } else if (OP == 4) {  // match.any on 13-bit values
        acc += __match_any_sync(0xffffffffu, ia) ^ __match_any_sync(0xffffffffu, ib) ^
               __match_any_sync(0xffffffffu, ic) ^ __match_any_sync(0xffffffffu, id);
      } else if (OP == 5) {  // ATOMS.ADD with return, per-warp private 256-word region
        const uint32_t base = (t >> 5) * 256;
        acc += atomicAdd(&s[base + (ia & 255)], 1u); acc += atomicAdd(&s[base + (ib & 255)], 1u);
        acc += atomicAdd(&s[base + (ic & 255)], 1u); acc += atomicAdd(&s[base + (id & 255)], 1u);
      } else if (OP == 6) {  // ATOMS.ADD conflict-free (lane-consecutive words)
        const uint32_t base = ((t >> 5) * 32 + (t & 31));
        acc += atomicAdd(&s[base + ((ia & 7) << 9)], 1u); acc += atomicAdd(&s[base + ((ib & 7) << 9)], 1u);
        acc += atomicAdd(&s[base + ((ic & 7) << 9)], 1u); acc += atomicAdd(&s[base + ((id & 7) << 9)], 1u);
      } else if (OP == 7) {  // STS conflict-free
        const uint32_t base = (t & 31);
        s[base + ((ia & 255) << 5)] = a; s[base + ((ib & 255) << 5)] = b;
        s[base + ((ic & 255) << 5)] = c; s[base + ((id & 255) << 5)] = d;
      } else if (OP == 8) {  // baseline: the LCG + shift only (ALU cost of address generation)
        acc += ia ^ ib ^ ic ^ id;
      }
    }
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + t] = acc + a + s[t];
  if (t == 0) out[gridDim.x * blockDim.x + blockIdx.x] = (uint32_t)(t1 - t0);
}

template <int OP>
void run(const char* name, int nthreads, int ctas_per_sm) {
  uint32_t* d;
  const int grid = 148 * ctas_per_sm;
  cudaMalloc(&d, (size_t(grid) * 1024 + grid) * 4);
  const size_t smem = TBL * 2 * 4;
  cudaFuncSetAttribute(k<OP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k<OP><<<grid, nthreads, smem>>>(d, 1);
  cudaDeviceSynchronize();
  k<OP><<<grid, nthreads, smem>>>(d, 2);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("%s: %s\n", name, cudaGetErrorString(e)); return; }
  uint32_t cyc;
  cudaMemcpy(&cyc, d + size_t(grid) * nthreads, 4, cudaMemcpyDeviceToHost);
  double warps = nthreads / 32.0 * ctas_per_sm;
  double instr = warps * ITERS * UNROLL * 4;  // per SM
  printf("%-34s %4d thr x %d CTA/SM: %7.3f clk per warp-instr per SM\n", name, nthreads, ctas_per_sm, cyc / instr);
  cudaFree(d);
}

int main() {
  for (int nt : {256, 512}) {
    for (int c : {1, 2}) {
      run<8>("baseline (address ALU only)", nt, c);
      run<0>("ATOMS.ADD ret, random 8K", nt, c);
      run<1>("RED.shared.ADD, random 8K", nt, c);
      run<2>("STS random 8K", nt, c);
      run<3>("LDS random 8K", nt, c);
      run<4>("MATCH.ANY 13-bit", nt, c);
      run<5>("ATOMS.ADD ret, per-warp 256", nt, c);
      run<6>("ATOMS.ADD ret, conflict-free", nt, c);
      run<7>("STS conflict-free", nt, c);
    }
  }
  return 0;
}
