// Instruction-throughput microbenchmarks on B200 (sm_100a): cycles per warp
// instruction per SM for the ops the sort kernels are made of.  Not part of the
// product; informs the kernel design.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define ITERS 4096
#define UNROLL 16

template <int OP>
__global__ void k(uint32_t* out, uint32_t seed) {
  __shared__ uint32_t s[8192 + 256];
  const int t = threadIdx.x;
  for (int i = t; i < 8192 + 256; i += blockDim.x) s[i] = i * 2654435761u;
  __syncthreads();
  uint32_t a = seed ^ t, b = t * 7 + 1, c = t * 13 + 5, d = t * 31 + 3;
  uint32_t e = a ^ 0x55, f = b ^ 0x77, g = c ^ 0x99, h = d ^ 0x11;
  long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int u = 0; u < UNROLL; u++) {
      if (OP == 0) {  // VIMNMX (min) 8 independent chains
        a = min(a, b ^ u); b = min(b, c ^ u); c = min(c, d ^ u); d = min(d, a ^ u);
        e = max(e, f ^ u); f = max(f, g ^ u); g = max(g, h ^ u); h = max(h, e ^ u);
      } else if (OP == 1) {  // IMAD
        a = a * b + c; b = b * c + d; c = c * d + e; d = d * e + f;
        e = e * f + g; f = f * g + h; g = g * h + a; h = h * a + b;
      } else if (OP == 2) {  // SHFL
        a = __shfl_xor_sync(0xffffffffu, a, 1); b = __shfl_xor_sync(0xffffffffu, b, 2);
        c = __shfl_xor_sync(0xffffffffu, c, 4); d = __shfl_xor_sync(0xffffffffu, d, 8);
        e = __shfl_xor_sync(0xffffffffu, e, 16); f = __shfl_xor_sync(0xffffffffu, f, 3);
        g = __shfl_xor_sync(0xffffffffu, g, 5); h = __shfl_xor_sync(0xffffffffu, h, 7);
      } else if (OP == 3) {  // LDS conflict-free (lane-consecutive)
        a += s[(t & 31) + ((a & 7) << 5)]; b += s[(t & 31) + 256 + ((b & 7) << 5)];
        c += s[(t & 31) + 512 + ((c & 7) << 5)]; d += s[(t & 31) + 768 + ((d & 7) << 5)];
        e += s[(t & 31) + 1024 + ((e & 7) << 5)]; f += s[(t & 31) + 1280 + ((f & 7) << 5)];
        g += s[(t & 31) + 1536 + ((g & 7) << 5)]; h += s[(t & 31) + 1792 + ((h & 7) << 5)];
      } else if (OP == 4) {  // LDS random addresses
        a += s[(a * 2654435761u) >> 19]; b += s[(b * 2654435761u) >> 19];
        c += s[(c * 2654435761u) >> 19]; d += s[(d * 2654435761u) >> 19];
        e += s[(e * 2654435761u) >> 19]; f += s[(f * 2654435761u) >> 19];
        g += s[(g * 2654435761u) >> 19]; h += s[(h * 2654435761u) >> 19];
      } else if (OP == 5) {  // SEL via ternary on predicate (ISETP + SEL pairs)
        a = (a < b) ? c : d; b = (b < c) ? d : e; c = (c < d) ? e : f; d = (d < e) ? f : g;
        e = (e < f) ? g : h; f = (f < g) ? h : a; g = (g < h) ? a : b; h = (h < a) ? b : c;
      } else if (OP == 6) {  // match.any
        a += __match_any_sync(0xffffffffu, a & 31); b += __match_any_sync(0xffffffffu, b & 31);
        c += __match_any_sync(0xffffffffu, c & 31); d += __match_any_sync(0xffffffffu, d & 31);
        e += __match_any_sync(0xffffffffu, e & 31); f += __match_any_sync(0xffffffffu, f & 31);
        g += __match_any_sync(0xffffffffu, g & 31); h += __match_any_sync(0xffffffffu, h & 31);
      } else if (OP == 7) {  // ballot + popc
        a += __popc(__ballot_sync(0xffffffffu, a & 1)); b += __popc(__ballot_sync(0xffffffffu, b & 1));
        c += __popc(__ballot_sync(0xffffffffu, c & 1)); d += __popc(__ballot_sync(0xffffffffu, d & 1));
        e += __popc(__ballot_sync(0xffffffffu, e & 1)); f += __popc(__ballot_sync(0xffffffffu, f & 1));
        g += __popc(__ballot_sync(0xffffffffu, g & 1)); h += __popc(__ballot_sync(0xffffffffu, h & 1));
      } else if (OP == 8) {  // LDS.128 conflict-free
        uint4 v0 = reinterpret_cast<const uint4*>(s)[(t & 31) + ((a & 7) << 5)];
        uint4 v1 = reinterpret_cast<const uint4*>(s)[(t & 31) + ((b & 7) << 5) + 256];
        a += v0.x ^ v0.w; b += v1.y ^ v1.z;
        uint4 v2 = reinterpret_cast<const uint4*>(s)[(t & 31) + ((c & 7) << 5) + 512];
        uint4 v3 = reinterpret_cast<const uint4*>(s)[(t & 31) + ((d & 7) << 5) + 768];
        c += v2.x ^ v2.w; d += v3.y ^ v3.z;
      } else if (OP == 9) {  // STS conflict-free
        s[(t & 31) + ((a & 7) << 5)] = b; s[(t & 31) + 256 + ((b & 7) << 5)] = c;
        s[(t & 31) + 512 + ((c & 7) << 5)] = d; s[(t & 31) + 768 + ((d & 7) << 5)] = a;
        a += 3; b += 5; c += 7; d += 11;
      } else if (OP == 10) {  // __vibmin (DPX): min + predicate
        bool p0, p1, p2, p3;
        a = __vibmin_u32(a, b ^ u, &p0); b = __vibmin_u32(b, c ^ u, &p1);
        c = __vibmin_u32(c, d ^ u, &p2); d = __vibmin_u32(d, a ^ u, &p3);
        e += p0; f += p1; g += p2; h += p3;
      }
    }
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + t] = a + b + c + d + e + f + g + h;
  if (t == 0) out[gridDim.x * blockDim.x + blockIdx.x] = (uint32_t)(t1 - t0);
}

template <int OP>
void run(const char* name, int nthreads, int perop) {
  uint32_t* d;
  cudaMalloc(&d, (148 * 1024 + 148) * 4);
  k<OP><<<148, nthreads>>>(d, 1);
  cudaDeviceSynchronize();
  k<OP><<<148, nthreads>>>(d, 2);
  cudaDeviceSynchronize();
  uint32_t cyc;
  cudaMemcpy(&cyc, d + 148 * nthreads, 4, cudaMemcpyDeviceToHost);
  double warps = nthreads / 32.0;
  double instr = warps * ITERS * UNROLL * perop;  // per SM
  printf("%-28s threads %4d: %8.3f warp-instr/clk/SM (%.2f cyc per warp-instr per SMSP)\n", name, nthreads,
         instr / cyc, cyc / (instr / 4));
  cudaFree(d);
}

int main() {
  for (int nt : {512, 1024}) {
    run<0>("VIMNMX", nt, 8);
    run<1>("IMAD", nt, 8);
    run<2>("SHFL", nt, 8);
    run<3>("LDS conflict-free", nt, 8);
    run<4>("LDS random", nt, 8);
    run<5>("ISETP+SEL", nt, 16);
    run<6>("MATCH.ANY", nt, 8);
    run<7>("VOTE.BALLOT+POPC", nt, 8);
    run<8>("LDS.128 conflict-free", nt, 4);
    run<9>("STS conflict-free", nt, 4);
    run<10>("VIBMIN (DPX)", nt, 4);
  }
  return 0;
}
