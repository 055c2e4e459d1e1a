// Microbenchmark: TMEM load (tcgen05.ld.32x32b) throughput per SM with 4..16
// warps, x8 / x16 / x32 shapes, one wait per load vs one wait per 4 loads.
#include <cstdio>
#include <cstdint>
#include "../../paper_2208_04448_b200/csrc/ptx.cuh"
using namespace nvdb;

__device__ __forceinline__ void ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

template <int SHAPE, int BATCH>
__global__ void k(int iters, long long* out, float* sink) {
  __shared__ uint32_t tslot;
  if (threadIdx.x < 32) tmem_alloc(&tslot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tslot + ((uint32_t)((threadIdx.x >> 5) & 3) * 32 << 16) + ((threadIdx.x >> 7) * 32);
  float acc = 0.f;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int b = 0; b < BATCH; ++b) {
      if (SHAPE == 8) { float v[8]; tmem_ld8(tm + b * 8, v); if (BATCH == 1) tmem_ld_wait(); acc += v[0] + v[7]; }
      if (SHAPE == 16) { float v[16]; tmem_ld16(tm + b * 16, v); if (BATCH == 1) tmem_ld_wait(); acc += v[0] + v[15]; }
      if (SHAPE == 32) { float v[32]; ld32(tm + b * 32, v); if (BATCH == 1) tmem_ld_wait(); acc += v[0] + v[31]; }
    }
    if (BATCH > 1) tmem_ld_wait();
  }
  __syncthreads();
  long long t1 = clock64();
  sink[threadIdx.x] = acc;
  if (threadIdx.x == 0) out[0] = t1 - t0;
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(tslot, 512);
}

template <int SHAPE, int BATCH>
void run(int warps, long long* d, float* sink) {
  const int iters = 2000;
  k<SHAPE, BATCH><<<1, warps * 32>>>(iters, d, sink);
  k<SHAPE, BATCH><<<1, warps * 32>>>(iters, d, sink);
  long long c;
  cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  const double bytes = (double)iters * BATCH * SHAPE * 4 * 32 * warps;
  printf("warps %2d x%-2d batch %d: %.1f B/clk per SM  (%s)\n", warps, SHAPE, BATCH, bytes / c,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  long long* d; float* sink;
  cudaMalloc(&d, 64); cudaMalloc(&sink, 4096 * 4);
  for (int w : {4, 8, 12, 16}) {
    run<16, 1>(w, d, sink);
    run<16, 3>(w, d, sink);
    run<8, 4>(w, d, sink);
    run<32, 2>(w, d, sink);
  }
  return 0;
}
