// Microbenchmark: tcgen05.mma (kind::f16, cta_group::1, M = 128) issue and
// execution rate from one thread, for several N, SS and TS operand modes.
#include <cstdio>
#include <cstdint>
#include "../../paper_2208_04448_b200/csrc/ptx.cuh"
using namespace nvdb;

__global__ void k(int N, int iters, int ts, int nd, long long* out, int noise) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (threadIdx.x < 32) tmem_alloc(&tslot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tslot;
  if (threadIdx.x >= 32 && noise) {
    // other warps: shared-memory store traffic (noise 1) or MUFU (noise 2) for ~ the same time
    const uint32_t base = smem_addr(smem + 131072) + (threadIdx.x & 255) * 16;
    float v = threadIdx.x;
    long long s0 = clock64();
    for (int i = 0; i < iters * 4; ++i) {
      if (noise == 1) st_shared_v4(base + (i & 15) * 4096, i, i, i, i);
      else v = __sinf(v);
    }
    if (v == 12345.f) out[7] = 1;
    if ((threadIdx.x & 31) == 0) out[16 + (threadIdx.x >> 5)] = clock64() - s0;
  }
  if (threadIdx.x == 0 && !(noise & 4)) {
    const uint32_t a = smem_addr(smem), b = smem_addr(smem + 65536);
    const uint32_t idesc = idesc_f16(128, N, 0, 0);
    const uint64_t ad = smem_desc(a, 128 * 16, 128), bd = smem_desc(b, N * 16, 128);
    long long t0 = clock64();
    if (ts) {
      for (int i = 0; i < iters; i += 4) {
        umma_f16_ts(tm, tm + 256, bd, idesc, 1);
        umma_f16_ts(tm, tm + 264, bd + 16, idesc, 1);
        umma_f16_ts(tm, tm + 272, bd + 32, idesc, 1);
        umma_f16_ts(tm, tm + 280, bd + 48, idesc, 1);
      }
    } else if (nd == 1) {
      for (int i = 0; i < iters; i += 4) {
        umma_f16(tm, ad, bd, idesc, 1);
        umma_f16(tm, ad + 256, bd + 16, idesc, 1);
        umma_f16(tm, ad + 512, bd + 32, idesc, 1);
        umma_f16(tm, ad + 768, bd + 48, idesc, 1);
      }
    } else {
      for (int i = 0; i < iters; i += 4) {
        umma_f16(tm, ad, bd, idesc, 1);
        umma_f16(tm + 128, ad + 256, bd + 16, idesc, 1);
        umma_f16(tm, ad + 512, bd + 32, idesc, 1);
        umma_f16(tm + 128, ad + 768, bd + 48, idesc, 1);
      }
    }
    long long t1 = clock64();
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t2 = clock64();
    out[0] = t1 - t0;
    out[1] = t2 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(tm, 512);
}

int main() {
  long long* d; cudaMalloc(&d, 256);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int noise : {0, 1, 5, 2, 6})
  for (int nd : {1})
  for (int ts = 0; ts < 2; ++ts)
    for (int N : {96}) {
      if (ts) continue;
      if (ts && nd > 1) continue;
      const int iters = 2048;
      k<<<1, 512, 200 * 1024>>>(N, iters, ts, nd, d, noise);
      k<<<1, 512, 200 * 1024>>>(N, iters, ts, nd, d, noise);
      long long h[32]; cudaMemcpy(h, d, 256, cudaMemcpyDeviceToHost);
      if (noise) {
        printf("  noise warps (%s, %s MMAs), clk per op: ", (noise & 3) == 1 ? "STS.128" : "MUFU", (noise & 4) ? "without" : "with");
        for (int w = 1; w < 16; ++w) printf("w%d:%.1f ", w, (double)h[16 + w] / (iters * 4));
        printf("\n");
      }
      cudaError_t e = cudaGetLastError();
      printf("noise=%d nd=%d %s N=%3d:", noise, nd, ts ? "TS" : "SS", N); printf(" issue %.1f clk/mma, complete %.1f clk/mma (ideal 128*N/256 = %d)  %s\n", (double)h[0] / iters, (double)h[1] / iters, 128 * N / 256, cudaGetErrorString(e));
    }
  return 0;
}
