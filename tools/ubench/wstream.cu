// Microbenchmark: the streamed-weight MMA loop of mlp_eval_kernel in
// isolation.  One CTA per SM, one issuing thread: a ring of WR slots of
// PIECES K = 16 weight chunks (W x 32 bytes each) filled by 1-D bulk copies
// from an L2-resident weight image, one tcgen05.mma (M = 128, N = W, K = 16)
// per chunk, one tcgen05.commit per slot to free it.  Reports clocks per
// K = 16 chunk for several ring depths / slot sizes.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o wstream wstream.cu && ./wstream
#include <cstdint>
#include <cstdio>
#include "../../paper_2208_04448_b200/csrc/ptx.cuh"
using namespace nvdb;

constexpr int W = 256;

// four K = 16 MMAs (B advancing by bstep, A by astep) in one asm block: one
// ELECT / R2UR sequence for the group instead of one per MMA
__device__ __forceinline__ void umma_f16_x4(uint32_t d, uint64_t ad, uint64_t bd, uint32_t idesc, uint32_t acc,
                                            uint64_t astep, uint64_t bstep) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t.reg .b64 a1, a2, a3, b1, b2, b3;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "add.u64 a1, %1, %5;\n\tadd.u64 a2, a1, %5;\n\tadd.u64 a3, a2, %5;\n\t"
      "add.u64 b1, %2, %6;\n\tadd.u64 b2, b1, %6;\n\tadd.u64 b3, b2, %6;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], a1, b1, %3, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], a2, b2, %3, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], a3, b3, %3, 1;\n\t}" ::"r"(d),
      "l"(ad), "l"(bd), "r"(idesc), "r"(acc), "l"(astep), "l"(bstep)
      : "memory");
}
constexpr uint32_t kChunk = W * 32;  // one K = 16 chunk

__global__ void __launch_bounds__(128, 1) k(const uint8_t* __restrict__ wimg, uint32_t nchunks, int WR, int PIECES,
                                            int iters, int AHEAD, int MODE, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t full[16], empty[16];
  __shared__ uint32_t tslot;
  const uint32_t slot_bytes = kChunk * PIECES;
  uint8_t* ring = smem + 32768;  // A tile (128 x 16 fp16 = 4 KB used) at 0
  if (threadIdx.x == 0) {
    for (int i = 0; i < 16; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    fence_barrier_init();
  }
  if (threadIdx.x < 32) tmem_alloc(&tslot, 512);
  for (int i = threadIdx.x; i < 8192; i += 128) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;  // A = ones
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (MODE == 6 && threadIdx.x == 32) {  // producer: refills each slot once its previous MMAs completed
    const uint32_t nslots_total = (uint32_t)iters * nchunks / PIECES;
    for (uint32_t pos = 0; pos < nslots_total; ++pos) {
      const uint32_t s = pos % WR;
      if (pos >= (uint32_t)WR) mbar_wait(&empty[s], ((pos / WR) - 1) & 1u);
      const uint32_t c = (pos * PIECES) % nchunks;
      mbar_arrive_expect_tx(&full[s], slot_bytes);
      bulk_g2s(ring + s * slot_bytes, wimg + (size_t)c * kChunk, slot_bytes, &full[s]);
    }
  }
  if (threadIdx.x == 0) {
    const uint32_t idesc = idesc_f16(128, W, 0, 0);
    const uint64_t ad = smem_desc(smem_addr(smem), 128 * 16, 128);
    const uint32_t nslots_total = (uint32_t)iters * nchunks / PIECES;
    uint32_t filled = 0;
    auto fill = [&](uint32_t pos) {
      const uint32_t s = pos % WR;
      if (pos >= (uint32_t)WR) mbar_wait(&empty[s], ((pos / WR) - 1) & 1u);
      const uint32_t c = (pos * PIECES + (MODE == 4 ? blockIdx.x * 5u : 0u)) % nchunks;
      mbar_arrive_expect_tx(&full[s], slot_bytes);
      bulk_g2s(ring + s * slot_bytes, wimg + (size_t)c * kChunk, slot_bytes, &full[s]);
    };
    if (MODE != 6 && MODE != 11)
      for (; filled < (uint32_t)(MODE >= 5 ? WR : AHEAD) && filled < nslots_total; ++filled) fill(filled);
    const long long t0 = clock64();
    for (uint32_t pos = 0; pos < (MODE == 11 ? 0u : nslots_total); ++pos) {
      if (MODE < 5 && filled < nslots_total && filled <= pos + AHEAD) fill(filled++);
      const uint32_t s = pos % WR;
      if (MODE != 3 && MODE != 5 && MODE < 7) mbar_wait(&full[s], (pos / WR) & 1u);
      if (MODE != 1 && MODE != 10) tc_fence_after();
      for (int p = 0; p < PIECES; ++p)
        umma_f16(tslot, ad, smem_desc(smem_addr(ring + s * slot_bytes + p * kChunk), W * 16, 128), idesc,
                 pos | p ? 1u : 0u);
      if (MODE == 2) {  // commit every second slot, to both slots' barriers
        if (pos & 1) {
          umma_commit(&empty[(pos - 1) % WR]);
          umma_commit(&empty[s]);
        }
      } else if (MODE == 7 || MODE == 10) {  // no commits in the loop
      } else if (MODE == 9) {  // one commit per 4 MMAs
        if ((pos & 3) == 3) umma_commit(&empty[s]);
      } else {
        umma_commit(&empty[s]);
      }
    }
    if (MODE == 11) {  // lean issue loop: power-of-two ring, incremental indices, precomputed descriptors
      const int lg = __ffs(WR) - 1;
      const uint64_t bd0 = smem_desc(smem_addr(ring), W * 16, 128);
      const uint32_t dstep = slot_bytes >> 4, pstep = kChunk >> 4;
      uint32_t fpos = 0, fc = 0;  // next fill position and its chunk
      const uint32_t npos = nslots_total;
      const long long t2 = clock64();
      for (; fpos < (uint32_t)(AHEAD % 100); ++fpos) {
        const uint32_t sl = fpos & (WR - 1);
        mbar_arrive_expect_tx(&full[sl], slot_bytes);
        bulk_g2s(ring + sl * slot_bytes, wimg + (size_t)fc * kChunk, slot_bytes, &full[sl]);
        fc += PIECES; if (fc >= nchunks) fc -= nchunks;
      }
      long long acc[7] = {0, 0, 0, 0, 0, 0, 0};
      for (uint32_t pos = 0; pos < npos; ++pos) {
        long long c0 = clock64(), c1;
        if (fpos < npos) {
          const uint32_t sl = fpos & (WR - 1);
          if (fpos >= (uint32_t)WR) mbar_wait(&empty[sl], ((fpos >> lg) - 1) & 1u);
          c1 = clock64(); acc[0] += c1 - c0; c0 = c1;
          mbar_arrive_expect_tx(&full[sl], slot_bytes);
          c1 = clock64(); acc[1] += c1 - c0; c0 = c1;
          bulk_g2s(ring + sl * slot_bytes, wimg + (size_t)fc * kChunk, slot_bytes, &full[sl]);
          c1 = clock64(); acc[2] += c1 - c0; c0 = c1;
          fc += PIECES; if (fc >= nchunks) fc -= nchunks;
          ++fpos;
        }
        const uint32_t sl = pos & (WR - 1);
        mbar_wait(&full[sl], (pos >> lg) & 1u);
        c1 = clock64(); acc[3] += c1 - c0; c0 = c1;
        tc_fence_after();
        c1 = clock64(); acc[4] += c1 - c0; c0 = c1;
        uint64_t bd = bd0 + sl * dstep;
        if (AHEAD >= 100 && PIECES == 4) umma_f16_x4(tslot, ad, bd, idesc, 1u, 0, pstep);
        else
          for (int p = 0; p < PIECES; ++p, bd += pstep) umma_f16(tslot, ad, bd, idesc, 1u);
        c1 = clock64(); acc[5] += c1 - c0; c0 = c1;
        umma_commit(&empty[sl]);
        c1 = clock64(); acc[6] += c1 - c0; c0 = c1;
      }
      if (blockIdx.x == 0)
        for (int i = 0; i < 7; ++i) out[2 + i] = acc[i];
      umma_commit(&full[15]);
      mbar_wait(&full[15], 0);
      if (blockIdx.x == 0) out[1] = clock64() - t2;
    }
    if (MODE != 11) {
      umma_commit(&full[15]);
      mbar_wait(&full[15], 0);
    }
    const long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(tslot, 512);
}

int main() {
  const uint32_t nchunks = 64;  // 512 KB image (3x256/m256 has 64 K = 16 chunks)
  uint8_t* wimg;
  long long* out;
  cudaMalloc(&wimg, nchunks * kChunk);
  cudaMemset(wimg, 0, nchunks * kChunk);
  cudaMalloc(&out, 128);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const int iters = 64;
  // MODE 0: as mlp_eval; 1: no tcgen05 fence after the wait; 2: one commit per two slots;
  // 3: no wait on the full barrier (data race, timing only); 4: each CTA starts at another chunk
  int cfg[][4] = {{2, 4, 1, 11}, {2, 4, 101, 11}, {4, 4, 2, 11}, {4, 4, 102, 11}};
  for (auto& c : cfg) {
    const int WR = c[0], PIECES = c[1], AHEAD = c[2], MODE = c[3];
    for (int rep = 0; rep < 2; ++rep) {
      k<<<148, 128, 200 * 1024>>>(wimg, nchunks, WR, PIECES, iters, AHEAD, MODE, out);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        printf("error %s\n", cudaGetErrorString(e));
        return 1;
      }
    }
    long long h[2];
    cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
    const long long clk = MODE == 11 ? h[1] : h[0];
    if (MODE == 11) {
      long long g[7];
      cudaMemcpy(g, out + 2, 56, cudaMemcpyDeviceToHost);
      const double ns = (double)iters * nchunks / PIECES;
      printf("  per slot: empty wait %.0f, expect_tx %.0f, bulk issue %.0f, full wait %.0f, fence %.0f, %d mma %.0f, commit %.0f\n",
             g[0] / ns, g[1] / ns, g[2] / ns, g[3] / ns, g[4] / ns, PIECES, g[5] / ns, g[6] / ns);
    }
    printf("mode %d ring %2d slots x %d chunks, %2d filled ahead: %6.1f clk per K=16 chunk (MMA alone 128)\n",
           MODE, WR, PIECES, AHEAD, (double)clk / (iters * nchunks));
  }
  return 0;
}
