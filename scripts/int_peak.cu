// Integer-pipe peak microbenchmark ("measure IMAD and ALU
// throughput on the box first"): dependent-chain-free streams of IMAD,
// IMAD.HI, IMAD.WIDE.U32 and IADD3 per thread, enough warps to saturate every
// SMSP; reports ops per second for the whole GPU.  Built and driven by
// scripts/int_peak.py.
#include <cstdint>
#include <cuda_runtime.h>

template <int OP>
__global__ void __launch_bounds__(256) k_int(uint32_t* out, uint32_t seed, int iters) {
  uint32_t a[8], b = seed * 2654435761u + threadIdx.x, c = seed ^ 0x9E3779B9u;
  uint64_t w[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = b + i * 77u, w[i] = a[i];
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 16; ++r) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (OP == 0) a[i] = a[i] * b + c;              // IMAD
        if (OP == 1) a[i] = __umulhi(a[i], b) + c;     // IMAD.HI (+ add folded)
        if (OP == 2) w[i] = w[i] + (uint64_t)(uint32_t)w[i] * b;  // IMAD.WIDE.U32 (64-bit addend)
        if (OP == 3) a[i] = a[i] + a[(i + 1) & 7] + c;             // IADD3 (no foldable chain)
      }
    }
  }
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i] + (uint32_t)w[i] + (uint32_t)(w[i] >> 32);
  if (s == 0x12345678u) out[0] = s;  // keep the work alive
}

extern "C" float int_peak(int op, int blocks, int iters) {
  uint32_t* out;
  cudaMalloc(&out, 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto launch = [&]() {
    switch (op) {
      case 0: k_int<0><<<blocks, 256>>>(out, 7, iters); break;
      case 1: k_int<1><<<blocks, 256>>>(out, 7, iters); break;
      case 2: k_int<2><<<blocks, 256>>>(out, 7, iters); break;
      default: k_int<3><<<blocks, 256>>>(out, 7, iters); break;
    }
  };
  launch();
  cudaEventRecord(e0);
  launch();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaFree(out);
  return ms;
}
