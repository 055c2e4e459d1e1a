// Microbenchmark: throughput of MUFU sin / ex2 / tanh, FMA-pipe sine polynomial
// and F2FP on one SM (all 4 SMSPs), in clocks per warp-instruction per SMSP.
#include <cstdio>
#include <cuda_fp16.h>

template <int OP>
__global__ void k(float* out, int iters, long long* clk) {
  float v[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = threadIdx.x * 1e-3f + i;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) v[i] = __sinf(v[i]);
      if (OP == 1) v[i] = exp2f(v[i]) ;
      if (OP == 2) { float r; asm("tanh.approx.f32 %0, %1;" : "=f"(r) : "f"(v[i])); v[i] = r; }
      if (OP == 3) { float r; asm("sin.approx.f32 %0, %1;" : "=f"(r) : "f"(v[i])); v[i] = r; }
      if (OP == 4) { float r; asm("ex2.approx.f32 %0, %1;" : "=f"(r) : "f"(v[i])); v[i] = r; }
      if (OP == 5) { __half2 h = __floats2half2_rn(v[i], v[(i+1)&7]); v[i] = __low2float(h) + 1.0f; }
      if (OP == 6) v[i] = fmaf(v[i], 1.0001f, 0.5f);
    }
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

int main() {
  float* out; long long* clk;
  cudaMalloc(&out, 1 << 20); cudaMalloc(&clk, 1024);
  const char* names[] = {"__sinf", "exp2f", "tanh.approx", "sin.approx", "ex2.approx", "F2FP+cvt+fadd", "FFMA"};
  for (int warps = 4; warps <= 32; warps *= 2) {
    for (int op = 0; op < 7; ++op) {
      const int iters = 4096;
      for (int rep = 0; rep < 2; ++rep) {
        switch (op) {
          case 0: k<0><<<1, warps * 32>>>(out, iters, clk); break;
          case 1: k<1><<<1, warps * 32>>>(out, iters, clk); break;
          case 2: k<2><<<1, warps * 32>>>(out, iters, clk); break;
          case 3: k<3><<<1, warps * 32>>>(out, iters, clk); break;
          case 4: k<4><<<1, warps * 32>>>(out, iters, clk); break;
          case 5: k<5><<<1, warps * 32>>>(out, iters, clk); break;
          case 6: k<6><<<1, warps * 32>>>(out, iters, clk); break;
        }
      }
      long long c; cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
      const double per_smsp_instr = (double)iters * 8 * warps / 4;
      printf("warps %2d %-16s %.2f clk per warp-op per SMSP (%.1f lanes/clk/SM)\n", warps, names[op],
             c / per_smsp_instr, 128.0 / (c / per_smsp_instr));
    }
  }
  return 0;
}
