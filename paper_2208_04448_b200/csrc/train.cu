// Device-resident training of one coordinate network (K4 + K5): the whole
// epoch loop of encoder.train_network (encoder.py:330-371) with
// neural.fused_step (neural.py:444-524) split into four kernels per epoch:
//
//   k_sample_*      numpy-exact batch indices: SeedSequence words (host) ->
//                   PCG64 jump-ahead -> buffered 32-bit Lemire (encoder.py:257-267)
//   k_train_fb      per 128-sample tile: gather, Fourier features, forward on
//                   tcgen05 (pre-activations kept in TMEM), fp32 head, loss and
//                   dL/dout, then the dgrad chain back to layer 0 on tcgen05
//                   (da = dz . W' with W' read as an MN-major operand).  Writes
//                   the fp16 activation / dz tiles the weight gradients need.
//   k_train_wgrad   weight gradients for every layer as tcgen05 GEMMs over the
//                   batch (split-K over CTAs, fp32 TMEM accumulators; bias
//                   gradients fall out of a ones column), per-CTA partials
//   k_train_adam    fixed-order reduction of the partials, bias-corrected Adam
//                   on fp32 master weights (numpy's op order and float32
//                   constants), refreshed fp16 weight image, batch loss,
//                   early stop flag; its last block advances the epoch.
//   (k_train_fb and k_train_wgrad run as one launch, k_train_fbwg, when they
//   share the tile partition.)
//
// Loss scaling: dL/dout is kept without the 1/size factor (fp16 would
// underflow at size 65536); the factor, and omega / amplitude folded into the
// fp16 weights, are applied in fp32 in the Adam kernel.
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <vector>

#include "netset.cuh"

#ifdef NVDB_TRACE
// trace build only: per-warp timeline of CTA 0 of the training kernels
__device__ unsigned long long* g_ttrace = nullptr;
__device__ unsigned int g_ttrace_cap = 0;
#define TTRC(ev, j)                                                                                \
  do {                                                                                             \
    if (blockIdx.x == 0 && g_ttrace && (threadIdx.x & 31) == 0 && ttrc_n < g_ttrace_cap) {         \
      unsigned long long* _r = g_ttrace + 2ull * ((threadIdx.x >> 5) * g_ttrace_cap + ttrc_n++);   \
      _r[0] = clock64();                                                                           \
      _r[1] = ((unsigned long long)(ev) << 32) | ((unsigned)(j) << 8) | (unsigned)(threadIdx.x >> 5); \
    }                                                                                              \
  } while (0)
#define TTRC_DECL unsigned int ttrc_n = 0
extern "C" __attribute__((visibility("default"))) int nvdb_debug_ttrace(void* buf, uint32_t cap) {
  unsigned long long* p = static_cast<unsigned long long*>(buf);
  cudaMemcpyToSymbol(g_ttrace, &p, sizeof(p));
  cudaMemcpyToSymbol(g_ttrace_cap, &cap, sizeof(cap));
  return cudaDeviceSynchronize() == cudaSuccess ? 0 : -2;
}
#else
#define TTRC(ev, j) \
  do {              \
  } while (0)
#define TTRC_DECL
#endif

using namespace nvdb;

namespace {

typedef unsigned __int128 u128;

// ------------------------------------------------------------------ sampler
__device__ __forceinline__ u128 pcg_mult() {
  return ((u128)0x2360ED051FC65DA4ULL << 64) | (u128)0x4385DF649FCCF645ULL;
}

// state after `delta` LCG steps (pcg_advance_lcg_128)
__device__ u128 pcg_advance(u128 state, u128 inc, unsigned long long delta) {
  u128 cur_mult = pcg_mult(), cur_plus = inc, acc_mult = 1, acc_plus = 0;
  while (delta > 0) {
    if (delta & 1ull) {
      acc_mult *= cur_mult;
      acc_plus = acc_plus * cur_mult + cur_plus;
    }
    cur_plus = (cur_mult + 1) * cur_plus;
    cur_mult *= cur_mult;
    delta >>= 1;
  }
  return acc_mult * state + acc_plus;
}

__device__ __forceinline__ unsigned long long pcg_out(u128 s) {
  const unsigned long long hi = (unsigned long long)(s >> 64), lo = (unsigned long long)s;
  const unsigned rot = (unsigned)(s >> 122);
  const unsigned long long x = hi ^ lo;
  return (x >> rot) | (x << ((64 - rot) & 63));
}

// PCG64 seeded from SeedSequence.generate_state(4, uint64) words
__device__ __forceinline__ void pcg_seed(const unsigned long long* w, u128& state, u128& inc) {
  const u128 initstate = ((u128)w[0] << 64) | (u128)w[1];
  const u128 initseq = ((u128)w[2] << 64) | (u128)w[3];
  inc = (initseq << 1) | 1;
  state = 0;
  state = state * pcg_mult() + inc;
  state += initstate;
  state = state * pcg_mult() + inc;
}

struct SampCtl {
  const int32_t* epoch;
  const int32_t* stopped;
  const unsigned long long* words;  // [max_epochs][4]
  unsigned long long n;             // draw range [0, n)
  int64_t batch;
  int64_t nraw;
  int32_t* flag;
  uint32_t* val;
  int32_t* pos;
  int64_t* idx;
};

__global__ void k_sample_raw(SampCtl c) {
  if (*c.stopped) return;
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t j0 = t * 8;
  if (j0 >= c.nraw) return;
  u128 st, inc;
  pcg_seed(c.words + 4 * (int64_t)(*c.epoch), st, inc);
  st = pcg_advance(st, inc, (unsigned long long)(j0 >> 1));
  const uint32_t nn = (uint32_t)c.n;
  const uint32_t threshold = (uint32_t)(0u - nn) % nn;
#pragma unroll
  for (int d = 0; d < 4; ++d) {
    st = st * pcg_mult() + inc;
    const unsigned long long o = pcg_out(st);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t j = j0 + 2 * d + h;
      if (j < c.nraw) {
        const uint32_t r = h ? (uint32_t)(o >> 32) : (uint32_t)o;
        const unsigned long long m = (unsigned long long)r * nn;
        c.flag[j] = ((uint32_t)m >= threshold) ? 1 : 0;
        c.val[j] = (uint32_t)(m >> 32);
      }
    }
  }
}

__global__ void k_sample_compact(SampCtl c) {
  if (*c.stopped) return;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < c.nraw; j += stride)
    if (c.flag[j] && c.pos[j] < c.batch) c.idx[c.pos[j]] = (int64_t)c.val[j];
}

// serial continuation if the parallel window had too many rejections
__global__ void k_sample_tail(SampCtl c) {
  if (*c.stopped || threadIdx.x != 0 || blockIdx.x != 0) return;
  int64_t have = c.pos[c.nraw - 1] + c.flag[c.nraw - 1];
  if (have >= c.batch) return;
  u128 st, inc;
  pcg_seed(c.words + 4 * (int64_t)(*c.epoch), st, inc);
  int64_t j = c.nraw;
  st = pcg_advance(st, inc, (unsigned long long)(j >> 1));
  unsigned long long o = 0;
  if (j & 1) o = pcg_out(st);  // high half of the draw whose low half was used
  const uint32_t nn = (uint32_t)c.n;
  const uint32_t threshold = (uint32_t)(0u - nn) % nn;
  while (have < c.batch) {
    uint32_t r;
    if ((j & 1) == 0) {
      st = st * pcg_mult() + inc;
      o = pcg_out(st);
      r = (uint32_t)o;
    } else {
      r = (uint32_t)(o >> 32);
    }
    ++j;
    const unsigned long long m = (unsigned long long)r * nn;
    if ((uint32_t)m >= threshold) c.idx[have++] = (int64_t)(m >> 32);
  }
}

// All epochs of a run at once: one CTA per epoch reproduces the numpy stream of
// Sampler.indices(epoch) (encoder.py:257-267) -- the same PCG64 / Lemire
// draws as k_sample_raw + scan + compact + tail -- into idx_all[epoch][batch]
// (int32).  Two passes per thread over its contiguous window of raw draws:
// count the accepted ones, block-wide exclusive scan, regenerate and write.
constexpr int kSampThreads = 1024;
// With a working subset (sample_interval > 1, encoder.py:260-267): the draws
// of epoch e are in [0, interval*batch) and map through subset[e / interval].
__global__ void __launch_bounds__(kSampThreads) k_sample_epochs(const unsigned long long* __restrict__ words,
                                                                 unsigned long long n, int64_t batch, int64_t nraw,
                                                                 int32_t e_begin, int32_t* __restrict__ idx_all,
                                                                 const int32_t* __restrict__ subset = nullptr,
                                                                 int64_t subset_len = 0, int32_t interval = 1) {
  typedef cub::BlockScan<int, kSampThreads> Scan;
  __shared__ typename Scan::TempStorage scan_tmp;
  __shared__ int s_total;
  const int e = e_begin + blockIdx.x;
  int32_t* out = idx_all + (int64_t)e * batch;
  const int32_t* sub = subset ? subset + (int64_t)(e / interval) * subset_len : nullptr;
  const uint32_t nn = (uint32_t)n;
  const uint32_t threshold = (uint32_t)(0u - nn) % nn;
  // window of raw draws per thread, even so a draw pair (one PCG output) never straddles two threads
  const int64_t per = ((nraw + kSampThreads - 1) / kSampThreads + 1) & ~1ll;
  const int64_t j0 = (int64_t)threadIdx.x * per, j1 = min(nraw, j0 + per);
  u128 st0, inc;
  pcg_seed(words + 4 * (int64_t)e, st0, inc);
  const u128 st_start = j0 < j1 ? pcg_advance(st0, inc, (unsigned long long)(j0 >> 1)) : st0;
  int cnt = 0;
  {
    u128 st = st_start;
    for (int64_t j = j0; j < j1; j += 2) {
      st = st * pcg_mult() + inc;
      const unsigned long long o = pcg_out(st);
      cnt += ((uint32_t)((unsigned long long)(uint32_t)o * nn) >= threshold) ? 1 : 0;
      if (j + 1 < j1) cnt += ((uint32_t)((unsigned long long)(uint32_t)(o >> 32) * nn) >= threshold) ? 1 : 0;
    }
  }
  int off, total;
  Scan(scan_tmp).ExclusiveSum(cnt, off, total);
  {
    u128 st = st_start;
    for (int64_t j = j0; j < j1 && off < batch; j += 2) {
      st = st * pcg_mult() + inc;
      const unsigned long long o = pcg_out(st);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (h == 1 && j + 1 >= j1) break;
        const uint32_t r = h ? (uint32_t)(o >> 32) : (uint32_t)o;
        const unsigned long long m = (unsigned long long)r * nn;
        if ((uint32_t)m >= threshold && off < batch) out[off++] = sub ? sub[m >> 32] : (int32_t)(m >> 32);
      }
    }
  }
  if (threadIdx.x == 0) s_total = total;
  __syncthreads();
  // serial continuation if the window had too many rejections (k_sample_tail)
  if (threadIdx.x == 0 && s_total < batch) {
    int64_t have = s_total, j = nraw;
    u128 st = pcg_advance(st0, inc, (unsigned long long)(j >> 1));
    unsigned long long o = 0;
    if (j & 1) o = pcg_out(st);
    while (have < batch) {
      uint32_t r;
      if ((j & 1) == 0) {
        st = st * pcg_mult() + inc;
        o = pcg_out(st);
        r = (uint32_t)o;
      } else {
        r = (uint32_t)(o >> 32);
      }
      ++j;
      const unsigned long long m = (unsigned long long)r * nn;
      if ((uint32_t)m >= threshold) out[have++] = sub ? sub[m >> 32] : (int32_t)(m >> 32);
    }
  }
}

// raw draws that cover `count` accepted bounded draws with margin (the tail
// kernel / serial continuation handles the rare excess of rejections)
int64_t raw_draws(uint64_t bound, int64_t count) {
  const double p_rej = bound > 1 ? (double)((uint32_t)(0u - (uint32_t)bound) % (uint32_t)bound) / 4294967296.0 : 0.0;
  const int64_t nraw = count + (int64_t)std::ceil(count * p_rej * 2.0) + 1024;
  return (nraw + 7) / 8 * 8;
}

__global__ void k_i32_to_i64(const int32_t* __restrict__ a, int64_t n, int64_t* __restrict__ b) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) b[i] = a[i];
}

__global__ void k_sample_ones(SampCtl c) {  // n == 1: numpy fills with 0 without drawing
  if (*c.stopped) return;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < c.batch; j += stride) c.idx[j] = 0;
}

// ------------------------------------------------------------------ fwd + dgrad
struct FbArgs {
  NetDev net;                 // current fp16 image etc. (device pointers)
  const float* xs;            // (n,3) normalized inputs
  const float* ys;            // (n,) targets / labels as float
  const int64_t* idx;         // batch -> point (nullable: identity)
  const int32_t* idx_all;     // [max_epochs][batch] presampled indices (used when non-null)
  const int32_t* epoch;       // device epoch counter (row of idx_all)
  int64_t batch;
  int64_t tile_begin, tile_end;  // this rank's share of the batch tiles
  int32_t loss_kind;          // 0 mse, 1 ce, 2 bce
  int32_t nwg;
  uint16_t* act_img;          // [depth][ntiles][128*W] fp16 tile images
  uint16_t* dz_img;           // [depth][ntiles][128*W]
  uint16_t* dlt_img;          // [ntiles][128*16]
  uint16_t* feat_img;         // [ntiles][128*k0] fp16 Fourier features (the weight-gradient phase reads them)
  double* loss_part;          // [grid]
  const int32_t* stopped;
  uint32_t w_off, region_off, region_bytes, small_off, bar_off;
};

// tile-image traffic between the fwd/dgrad and weight-gradient phases: the
// images are written with L2 evict_last and read once with evict_first, so
// the most recent tiles (read first by the weight-gradient phase) stay in L2
#ifndef NVDB_L2HINT
#define NVDB_L2HINT 1
#endif
__device__ __forceinline__ void img_store(void* p, uint4 v, uint64_t pol) {
  if (NVDB_L2HINT) st_global_v4_hint(p, v, pol);
  else *reinterpret_cast<uint4*>(p) = v;
}
__device__ __forceinline__ void img_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  if (NVDB_L2HINT) bulk_g2s_hint(dst, src, bytes, bar, pol);
  else bulk_g2s(dst, src, bytes, bar);
}

__device__ __forceinline__ float act_deriv_from(int act, float zp) {
  if (act == ACT_SINE) return __cosf(zp);
  if (act == ACT_TANH) {
    const float a = tanhf(zp);
    return 1.0f - a * a;
  }
  return zp > 0.0f ? 1.0f : 0.0f;
}

__device__ __forceinline__ void fb_body(const FbArgs& a, uint8_t* smem) {
  TTRC_DECL;
  const int tid = threadIdx.x;
  const int grp = tid >> 8;               // tile group (a.nwg groups of 8 warps)
  const int gt = tid & 255;
  const int gw = gt >> 5;
  const int quad = gw & 3;                // TMEM lane quadrant
  const int half = gw >> 2;               // half of the feature pairs / columns
  const int row = quad * 32 + (gt & 31);  // tile row == TMEM lane
  const int nthreads = a.nwg * 256;
  const NetDev& nd = a.net;
  const int width = nd.width, depth = nd.depth, k0 = nd.k0, out_dim = nd.out_dim, act = nd.act;
  const int mp = k0 >> 1;
  uint8_t* wsm = smem + a.w_off;
  float* small = reinterpret_cast<float*>(smem + a.small_off);
  float* s_bias = small + kSmallBias;
  float* s_headw = small + kSmallHeadW;
  float* s_headb = small + kSmallHeadB;
  float* s_b2pi = small + kSmallB2pi;
  float* s_hx = small + kSmallHx + grp * 128 * 4;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + a.bar_off);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 8);
  __shared__ double s_loss[2][8];

  if (tid == 0) {
    for (int i = 0; i < 7; ++i) mbar_init(&bars[i], 1);
    fence_barrier_init();
    mbar_arrive_expect_tx(&bars[0], nd.wimg_bytes);
    for (uint32_t off = 0; off < nd.wimg_bytes; off += 32768)
      bulk_g2s(wsm + off, nd.wimg + off, min(32768u, nd.wimg_bytes - off), &bars[0]);
  }
  if (tid < 32) tmem_alloc_keep(tmem_slot, 512);
  for (int i = tid; i < depth * width; i += nthreads) s_bias[i] = nd.bias[i];
  for (int i = tid; i < out_dim * width; i += nthreads) s_headw[i] = nd.headw[i];
  if (tid < out_dim) s_headb[tid] = nd.headb[tid];
  for (int i = tid; i < 3 * mp; i += nthreads) s_b2pi[i] = nd.b2pi[i];
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  mbar_wait(&bars[0], 0);
  const uint32_t tmem_base = *tmem_slot;
  uint64_t* bar_c0 = &bars[1 + 3 * grp];
  uint64_t* bar_layer = &bars[3 + 3 * grp];
  uint32_t nc0 = 0, nc1 = 0, nlayer = 0;
  bool pend0 = false, pend1 = false;
  // per group: Z (W fp32 columns: every layer's accumulator in turn, then the
  // dgrad outputs) | F (depth x W/2 columns: f'(z_l) as fp16 pairs)
  const uint32_t tcol = tmem_base + (uint32_t)(grp * 256);
  const uint32_t fcol = tcol + (uint32_t)width;
  const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
  const uint32_t region_s = smem_addr(smem + a.region_off + grp * a.region_bytes);
  const uint32_t w_s = smem_addr(wsm);
  const uint32_t idesc = idesc_f16(kTileM, width, 0, 0);
  const uint32_t idesc_bt = idesc_f16(kTileM, width, 0, 1);  // B = W'^T read MN-major

  const int64_t ntiles = (a.batch + kTileM - 1) / kTileM;
  const int64_t per = (a.tile_end - a.tile_begin + gridDim.x - 1) / gridDim.x;
  const int64_t t0 = a.tile_begin + blockIdx.x * per, t1 = min(a.tile_end, t0 + per);
  double loss_acc = 0.0;
  const size_t tile_elems = (size_t)kTileM * width;
  const uint64_t pol_img = l2_evict_last();  // tile images: re-read by the weight-gradient phase

  // inputs of this thread's row, loaded one tile ahead (the gather through the
  // sampled indices is two dependent global loads)
  const int32_t* eidx = a.idx_all ? a.idx_all + (int64_t)(*a.epoch) * a.batch : nullptr;
  auto load_row = [&](int64_t tt, float& x0, float& x1, float& x2, float& y) {
    const int64_t bb = tt * kTileM + row;
    if (tt < t1 && bb < a.batch) {
      const int64_t pi = eidx ? (int64_t)eidx[bb] : (a.idx ? a.idx[bb] : bb);
      x0 = a.xs[3 * pi]; x1 = a.xs[3 * pi + 1]; x2 = a.xs[3 * pi + 2];
      y = a.ys[pi];
    } else {
      x0 = x1 = x2 = y = 0.f;
    }
  };
  float nx0, nx1, nx2, ny;
  load_row(t0 + grp, nx0, nx1, nx2, ny);
  for (int64_t tau = t0 + grp; tau < t1; tau += a.nwg) {
    const int64_t b = tau * kTileM + row;
    const bool valid = b < a.batch;
    const float x0 = nx0, x1 = nx1, x2 = nx2, y = ny;
    load_row(tau + a.nwg, nx0, nx1, nx2, ny);
    TTRC(1, tau);
    // ---------------- features + layer 0 (as in mlp_eval_kernel)
    const int nch = k0 / kChunkK;
    for (int ch = 0; ch < nch; ++ch) {
      const int bsel = ch & 1;
      if (bsel == 0 && pend0) { mbar_wait(bar_c0, (nc0 - 1u) & 1u); pend0 = false; }
      if (bsel == 1 && pend1) { mbar_wait(bar_c0 + 1, (nc1 - 1u) & 1u); pend1 = false; }
      const uint32_t buf = region_s + bsel * kChunkBytes;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint32_t h[4];
        const int f0 = ch * (kChunkK / 2) + half * 16 + q * 4;  // 4 features: one 16-byte load per axis
        const float4 bx = *reinterpret_cast<const float4*>(s_b2pi + f0);
        const float4 by = *reinterpret_cast<const float4*>(s_b2pi + mp + f0);
        const float4 bz = *reinterpret_cast<const float4*>(s_b2pi + 2 * mp + f0);
        const float bxa[4] = {bx.x, bx.y, bx.z, bx.w}, bya[4] = {by.x, by.y, by.z, by.w};
        const float bza[4] = {bz.x, bz.y, bz.z, bz.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float th = fmaf(x2, bza[j], fmaf(x1, bya[j], x0 * bxa[j]));
          float sn, cs;
          __sincosf(th, &sn, &cs);
          h[j] = pack_half2(cs, sn);
        }
        const uint32_t fo = kmajor_offset(row, half * 32 + q * 8, kTileM);
        st_shared_v4(buf + fo, h[0], h[1], h[2], h[3]);
        img_store(reinterpret_cast<uint8_t*>(a.feat_img) + (size_t)tau * kTileM * k0 * 2 + (size_t)ch * kChunkBytes + fo,
                  make_uint4(h[0], h[1], h[2], h[3]), pol_img);
      }
      fence_async_smem();
      tc_fence_before();
      named_bar_sync(1 + grp, 256);
      if (gw == 0) {  // the group's first warp issues converged (elect inside the asm)
        tc_fence_after();
        umma_f16_run_w(tcol, smem_desc(buf, kTileM * 16, 128),
                       smem_desc(w_s + (uint32_t)(((ch * kChunkK) >> 3) * (width >> 3) * 128), width * 16, 128),
                       idesc, ch != 0, kChunkK / 16, 256, (uint64_t)(width * 2));
        umma_commit_w(bar_c0 + bsel);
        if (ch == nch - 1) umma_commit_w(bar_layer);
      }
      if (bsel == 0) { nc0++; pend0 = true; } else { nc1++; pend1 = true; }
    }
    TTRC(2, tau);
    mbar_wait(bar_layer, nlayer & 1u);
    nlayer++;
    pend0 = pend1 = false;
    tc_fence_after();
    TTRC(3, tau);
    // ---------------- hidden layers: z_h stays in TMEM columns [h*W, (h+1)*W)
    float yv[3] = {0.f, 0.f, 0.f};
    uint32_t woff = (uint32_t)(width * k0 * 2);
    for (int l = 0; l < depth; ++l) {
      const bool last = (l == depth - 1);
      const float* bl = s_bias + l * width;
      uint16_t* gact = a.act_img + ((size_t)l * ntiles + tau) * tile_elems;
      // this thread's 16-column groups (cc = half, half + 2, ...), all TMEM loads first
      const int ncc = width / 16;
      const int nmine = (ncc - half + 1) / 2;
      for (int c0 = 0; c0 < nmine; c0 += 2) {
        const int nb = min(2, nmine - c0);
        float v[2][16];
#pragma unroll
        for (int b2 = 0; b2 < 2; ++b2)
          if (b2 < nb) tmem_ld16(tcol + lane_off + (half + 2 * (c0 + b2)) * 16, v[b2]);
        tmem_ld_wait();
#pragma unroll
        for (int b2 = 0; b2 < 2; ++b2) {
          if (b2 >= nb) break;
          const int cc = half + 2 * (c0 + b2);
          float av[16];
          uint32_t fpk[8];  // f'(z) for the backward pass, fp16 pairs -> TMEM F_l
#pragma unroll
          for (int i = 0; i < 16; i += 2) {
            const float2 bb = *reinterpret_cast<const float2*>(bl + cc * 16 + i);
            const float2 z = __fadd2_rn(make_float2(v[b2][i], v[b2][i + 1]), bb);
            if (act == ACT_SINE) {  // sin and cos of one argument (one range reduction)
              float c0, c1;
              __sincosf(z.x, &av[i], &c0);
              __sincosf(z.y, &av[i + 1], &c1);
              fpk[i >> 1] = pack_half2(c0, c1);
            } else {
              av[i] = act_fn(act, z.x);
              av[i + 1] = act_fn(act, z.y);
              fpk[i >> 1] = pack_half2(act_deriv_from(act, z.x), act_deriv_from(act, z.y));
            }
          }
          tmem_st8(fcol + (uint32_t)(l * (width >> 1)) + lane_off + cc * 8, fpk);
          const uint32_t p0 = pack_half2(av[0], av[1]), p1 = pack_half2(av[2], av[3]);
          const uint32_t p2 = pack_half2(av[4], av[5]), p3 = pack_half2(av[6], av[7]);
          const uint32_t p4 = pack_half2(av[8], av[9]), p5 = pack_half2(av[10], av[11]);
          const uint32_t p6 = pack_half2(av[12], av[13]), p7 = pack_half2(av[14], av[15]);
          const uint32_t o0 = kmajor_offset(row, cc * 16, kTileM), o1 = kmajor_offset(row, cc * 16 + 8, kTileM);
          img_store(reinterpret_cast<uint8_t*>(gact) + o0, make_uint4(p0, p1, p2, p3), pol_img);
          img_store(reinterpret_cast<uint8_t*>(gact) + o1, make_uint4(p4, p5, p6, p7), pol_img);
          if (!last) {
            st_shared_v4(region_s + o0, p0, p1, p2, p3);
            st_shared_v4(region_s + o1, p4, p5, p6, p7);
          } else {
#pragma unroll
            for (int k = 0; k < 3; ++k) {
              if (k < out_dim) {
                float sp[4];
#pragma unroll
                for (int q4 = 0; q4 < 4; ++q4) {  // four short partial sums
                  const float* hw = s_headw + k * width + cc * 16 + 4 * q4;
                  sp[q4] = fmaf(av[4 * q4], hw[0], av[4 * q4 + 1] * hw[1]);
                  sp[q4] = fmaf(av[4 * q4 + 2], hw[2], sp[q4]);
                  sp[q4] = fmaf(av[4 * q4 + 3], hw[3], sp[q4]);
                }
                yv[k] += (sp[0] + sp[1]) + (sp[2] + sp[3]);
              }
            }
          }
        }
      }
      tmem_st_wait();
      if (!last) {
        fence_async_smem();
        tc_fence_before();
        named_bar_sync(1 + grp, 256);
        if (gw == 0) {
          tc_fence_after();
          const uint32_t wl = w_s + woff;
          umma_f16_run_w(tcol, smem_desc(region_s, kTileM * 16, 128), smem_desc(wl, width * 16, 128), idesc, 0u,
                         width / 16, 256, (uint64_t)(width * 2));
          umma_commit_w(bar_layer);
        }
        woff += (uint32_t)(width * width * 2);
        mbar_wait(bar_layer, nlayer & 1u);
        nlayer++;
        tc_fence_after();
      }
    }
    TTRC(4, tau);
    // ---------------- head partials meet; loss and dL/dout (neural.py:271-302, without 1/size)
    if (half) {
#pragma unroll
      for (int k = 0; k < 3; ++k) s_hx[row * 4 + k] = yv[k];
    }
    named_bar_sync(1 + grp, 256);
    float dl[3] = {0.f, 0.f, 0.f};
    float lterm = 0.f;
    if (!half) {
#pragma unroll
      for (int k = 0; k < 3; ++k)
        if (k < out_dim) yv[k] = (yv[k] + s_hx[row * 4 + k]) + s_headb[k];
      if (valid) {
        if (a.loss_kind == 0) {  // mse
          const float d = yv[0] - y;
          lterm = d * d;
          dl[0] = 2.0f * d;
        } else if (a.loss_kind == 2) {  // bce
          const float z = yv[0];
          lterm = fmaxf(z, 0.f) - z * y + log1pf(expf(-fabsf(z)));
          dl[0] = 1.0f / (1.0f + expf(-z)) - y;
        } else {  // ce, 3 classes
          const float zm = fmaxf(fmaxf(yv[0], yv[1]), yv[2]);
          const float e0 = expf(yv[0] - zm), e1 = expf(yv[1] - zm), e2 = expf(yv[2] - zm);
          const float s = (e0 + e1) + e2;
          const int lab = (int)y;
          const float zl = lab == 0 ? yv[0] : (lab == 1 ? yv[1] : yv[2]);
          lterm = -(zl - zm - logf(s));
          dl[0] = e0 / s - (lab == 0 ? 1.f : 0.f);
          dl[1] = e1 / s - (lab == 1 ? 1.f : 0.f);
          dl[2] = e2 / s - (lab == 2 ? 1.f : 0.f);
        }
      }
      uint8_t* gd = reinterpret_cast<uint8_t*>(a.dlt_img + (size_t)tau * kTileM * 16);
      img_store(gd + kmajor_offset(row, 0, kTileM), make_uint4(pack_half2(dl[0], dl[1]), pack_half2(dl[2], 0.f), 0u, 0u),
                pol_img);
      img_store(gd + kmajor_offset(row, 8, kTileM), make_uint4(0u, 0u, 0u, 0u), pol_img);
    }
    // deterministic loss sum: warp shuffle, then fixed warp order
    float ls = lterm;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ls += __shfl_xor_sync(0xffffffffu, ls, o);
    if ((gt & 31) == 0) s_loss[grp][gw] = (double)ls;
    named_bar_sync(1 + grp, 256);  // also publishes the head partials' slots for reuse below
    if (gt == 0) loss_acc += ((s_loss[grp][0] + s_loss[grp][1]) + s_loss[grp][2]) + s_loss[grp][3];
    if (!half) {
#pragma unroll
      for (int k = 0; k < 3; ++k) s_hx[row * 4 + k] = dl[k];
    }
    named_bar_sync(1 + grp, 256);
    if (half) {
#pragma unroll
      for (int k = 0; k < 3; ++k) dl[k] = s_hx[row * 4 + k];
    }
    TTRC(5, tau);
    // ---------------- backward: dz_h = da_h * f'(z'_h); da_{h-1} = dz_h . W'_h
    for (int l = depth - 1; l >= 0; --l) {
      const float* bl = s_bias + l * width;
      uint16_t* gdz = a.dz_img + ((size_t)l * ntiles + tau) * tile_elems;
      const int ncc = width / 16;
      const int nmine = (ncc - half + 1) / 2;
      const bool top = (l == depth - 1);
      for (int c0 = 0; c0 < nmine; c0 += 1) {
        const int nb = 1;
        float fz[1][8], da[1][16];
#pragma unroll
        for (int b2 = 0; b2 < 1; ++b2) {
          if (b2 < nb) {
            const int cc = half + 2 * (c0 + b2);
            tmem_ld8(fcol + (uint32_t)(l * (width >> 1)) + lane_off + cc * 8, fz[b2]);
            if (!top) tmem_ld16(tcol + lane_off + cc * 16, da[b2]);
          }
        }
        tmem_ld_wait();
#pragma unroll
        for (int b2 = 0; b2 < 1; ++b2) {
          if (b2 >= nb) break;
          const int cc = half + 2 * (c0 + b2);
          if (top) {
#pragma unroll
            for (int i4 = 0; i4 < 4; ++i4) {
              float4 s4 = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
              for (int k = 0; k < 3; ++k) {
                if (k < out_dim) {
                  const float4 hw = *reinterpret_cast<const float4*>(s_headw + k * width + cc * 16 + 4 * i4);
                  s4.x = fmaf(dl[k], hw.x, s4.x);
                  s4.y = fmaf(dl[k], hw.y, s4.y);
                  s4.z = fmaf(dl[k], hw.z, s4.z);
                  s4.w = fmaf(dl[k], hw.w, s4.w);
                }
              }
              da[b2][4 * i4] = s4.x;
              da[b2][4 * i4 + 1] = s4.y;
              da[b2][4 * i4 + 2] = s4.z;
              da[b2][4 * i4 + 3] = s4.w;
            }
          }
          float dz[16];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const __half2 h = *reinterpret_cast<const __half2*>(&fz[b2][i]);
            const float2 f = __half22float2(h);
            const float2 d2 = __fmul2_rn(make_float2(da[b2][2 * i], da[b2][2 * i + 1]), f);
            dz[2 * i] = valid ? d2.x : 0.f;
            dz[2 * i + 1] = valid ? d2.y : 0.f;
          }
          const uint32_t p0 = pack_half2(dz[0], dz[1]), p1 = pack_half2(dz[2], dz[3]);
          const uint32_t p2 = pack_half2(dz[4], dz[5]), p3 = pack_half2(dz[6], dz[7]);
          const uint32_t p4 = pack_half2(dz[8], dz[9]), p5 = pack_half2(dz[10], dz[11]);
          const uint32_t p6 = pack_half2(dz[12], dz[13]), p7 = pack_half2(dz[14], dz[15]);
          const uint32_t o0 = kmajor_offset(row, cc * 16, kTileM), o1 = kmajor_offset(row, cc * 16 + 8, kTileM);
          img_store(reinterpret_cast<uint8_t*>(gdz) + o0, make_uint4(p0, p1, p2, p3), pol_img);
          img_store(reinterpret_cast<uint8_t*>(gdz) + o1, make_uint4(p4, p5, p6, p7), pol_img);
          if (l > 0) {
            st_shared_v4(region_s + o0, p0, p1, p2, p3);
            st_shared_v4(region_s + o1, p4, p5, p6, p7);
          }
        }
      }
      if (l > 0) {
        fence_async_smem();
        tc_fence_before();
        named_bar_sync(1 + grp, 256);
        if (gw == 0) {
          tc_fence_after();
          // W'_l image (rows o, cols i, K-major) read as B = (N = i, K = o) MN-major
          const uint32_t wl = w_s + (uint32_t)(width * k0 * 2) + (uint32_t)((l - 1) * width * width * 2);
          umma_f16_run_w(tcol, smem_desc(region_s, kTileM * 16, 128), smem_desc(wl, 128, width * 16), idesc_bt, 0u,
                         width / 16, 256, 16);
          umma_commit_w(bar_layer);
        }
        mbar_wait(bar_layer, nlayer & 1u);
        nlayer++;
        tc_fence_after();
      }
    }
    tc_fence_before();
    named_bar_sync(1 + grp, 256);  // all TMEM reads of this tile done before the next tile's MMAs
    TTRC(6, tau);
  }
  // per-CTA loss partial (fixed order: group 0 then group 1)
  __shared__ double s_wgl[2];
  if (gt == 0) s_wgl[grp] = loss_acc;
  tc_fence_before();
  __syncthreads();
  if (tid == 0) {
    a.loss_part[blockIdx.x] = a.nwg == 2 ? s_wgl[0] + s_wgl[1] : s_wgl[0];
    for (int i = 0; i < 7; ++i) mbar_inval(&bars[i]);
  }
  if (tid < 32) tmem_dealloc(tmem_base, 512);
}

__global__ void __launch_bounds__(512, 1) k_train_fb(const FbArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  if (*a.stopped) return;
  fb_body(a, smem);
}

// ------------------------------------------------------------------ weight gradients
constexpr uint32_t kWgSmem = 208896 + 3 * 512 * 4 + 128;

struct WgArgs {
  NetDev net;
  int32_t m;                  // real frequency count (2m real features)
  int32_t width_real;         // real hidden width
  const float* xs;
  const int64_t* idx;
  int64_t batch;
  int64_t tile_begin, tile_end;
  const uint16_t* act_img;
  const uint16_t* dz_img;
  const uint16_t* dlt_img;
  const uint16_t* feat_img;   // [ntiles][128*k0] written by the forward phase
  float* partial;             // [grid][P]
  int64_t P;
  const int64_t* poff;        // per layer l: offset of W_l, then of b_l ([2*(depth+1)])
  const int32_t* stopped;
  uint32_t col_w0, col_b0, col_h, col_head;  // TMEM column bases
  uint32_t col_hb;            // W > 112: per-layer bias gradients (16 columns each: hidden layers, then head)
  int32_t two_pass;           // accumulators exceed 512 TMEM columns: gW0 pass, then the rest
};

// mode 0: every accumulator in one pass over the tiles; when they exceed the
// 512 TMEM columns the host runs two passes: mode 1 = gW0 only (features x
// dz0), mode 2 = everything else, its columns shifted down by the gW0 block.
template <int mode>
__device__ __forceinline__ void wg_body(const WgArgs& a, uint8_t* smem) {
  TTRC_DECL;
#ifdef NVDB_TRACE
  ttrc_n = g_ttrace_cap / 2;  // after the fb records of the fused kernel
#endif
  const int t = threadIdx.x;
  const int row = t & 127;
  const int half = t >> 7;
  const int quad = (t >> 5) & 3;
  const NetDev& nd = a.net;
  const int W = nd.width, depth = nd.depth, k0 = nd.k0, mp = k0 >> 1;
  // smem: 2 x [act 32K | dz 32K] | feat ring 2 x 32K | 2 x dlt 4K | ones 4K | b2pi | bars
  uint8_t* s_act[2] = {smem, smem + 65536};
  uint8_t* s_dz[2] = {smem + 32768, smem + 65536 + 32768};
  uint8_t* s_feat = smem + 131072;
  uint8_t* s_dlt[2] = {smem + 196608, smem + 200704};
  uint8_t* s_ones = smem + 204800;
  float* s_b2pi = reinterpret_cast<float*>(smem + 208896);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 208896 + 3 * 512 * 4);
  // bars: [0,1] full (stage data landed), [2,3] free (stage MMAs done), [4,5] feature ring free, [6] final,
  // [7,8] feature chunk landed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 12);
  if (t == 0) {
    for (int i = 0; i < 9; ++i) mbar_init(&bars[i], 1);
    fence_barrier_init();
  }
  if (t < 32) tmem_alloc_keep(tmem_slot, 512);
  for (int i = t; i < 3 * mp; i += 256) s_b2pi[i] = nd.b2pi[i];
  for (int i = t; i < 16 * 128; i += 256) reinterpret_cast<__half*>(s_ones)[i] = __float2half(1.0f);
  // W <= 112: the bias gradients of hidden layers and head fall out of a ones
  // column appended to the activation operand (row W of [a | 1]^T); wider
  // layers fill all 128 rows, so their biases take separate MMAs (sep_bias)
  const bool sep_bias = W > kTileM - 16;
  if (t < 128 && !sep_bias) {  // ones column (W) and zero columns (W+1..W+15) of both augmented activation buffers
    for (int b = 0; b < 2; ++b) {
      const uint32_t o0 = kmajor_offset(t, W, kTileM), o1 = kmajor_offset(t, W + 8, kTileM);
      *reinterpret_cast<uint4*>(s_act[b] + o0) = make_uint4(pack_half2(1.f, 0.f), 0u, 0u, 0u);
      *reinterpret_cast<uint4*>(s_act[b] + o1) = make_uint4(0u, 0u, 0u, 0u);
    }
  }
  fence_async_smem();
  tc_fence_before();
  named_bar_sync(3, 256);
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
  const int64_t ntiles = (a.batch + kTileM - 1) / kTileM;
  const int64_t per = (a.tile_end - a.tile_begin + gridDim.x - 1) / gridDim.x;
  const int64_t t0 = a.tile_begin + blockIdx.x * per, t1 = min(a.tile_end, t0 + per);
  const size_t tbytes = (size_t)kTileM * W * 2;
  const uint64_t pol_rd = l2_evict_first();  // each tile image is read once
  const uint32_t sfe = smem_addr(s_feat), son = smem_addr(s_ones);
  const int nmt = (k0 + 127) / 128;  // M tiles of 128 features
  const int nst = mode == 1 ? 1 : depth + 1;  // load stages per tile: dz0 | (a0,dz1) .. | (a_{d-1}, dlt)
  const bool do_w0 = mode != 2, do_rest = mode != 1;
  const uint32_t sh = mode == 2 ? (uint32_t)(nmt * W) : 0u;  // mode 2: columns without the gW0 block
  const uint32_t col_b0 = a.col_b0 - sh, col_h = a.col_h - sh, col_head = a.col_head - sh, col_hb = a.col_hb - sh;
  const int64_t nstages = (t1 - t0) * nst;
  // thread-0 pipeline state
  uint32_t nfull[2] = {0, 0}, nfree[2] = {0, 0};
  bool busy[2] = {false, false};
  int64_t issued = 0;  // stages whose loads were issued
  uint32_t nring0 = 0, nring1 = 0, nfeat[2] = {0, 0};
  bool pr0 = false, pr1 = false;

  auto issue_load = [&](int64_t q) {  // thread 0 only
    const int b = (int)(q & 1);
    const int64_t tau = t1 - 1 - q / nst;  // newest tile first: the forward phase's latest images are L2-hot
    const int s = (int)(q % nst);
    if (busy[b]) {  // stage q-2 used this buffer: wait for its MMAs
      mbar_wait(&bars[2 + b], (nfree[b] - 1u) & 1u);
      busy[b] = false;
    }
    uint32_t bytes = (uint32_t)tbytes;
    if (s > 0) bytes += (s == depth) ? (uint32_t)(kTileM * 16 * 2) : (uint32_t)tbytes;
    mbar_arrive_expect_tx(&bars[b], bytes);
    if (s == 0) {
      img_load(s_dz[b], reinterpret_cast<const uint8_t*>(a.dz_img) + tau * tbytes, (uint32_t)tbytes, &bars[b], pol_rd);
    } else {
      img_load(s_act[b], reinterpret_cast<const uint8_t*>(a.act_img) + ((size_t)(s - 1) * ntiles + tau) * tbytes,
               (uint32_t)tbytes, &bars[b], pol_rd);
      if (s == depth)
        img_load(s_dlt[b], reinterpret_cast<const uint8_t*>(a.dlt_img) + (size_t)tau * kTileM * 16 * 2,
                 kTileM * 16 * 2, &bars[b], pol_rd);
      else
        img_load(s_dz[b], reinterpret_cast<const uint8_t*>(a.dz_img) + ((size_t)s * ntiles + tau) * tbytes,
                 (uint32_t)tbytes, &bars[b], pol_rd);
    }
  };
  auto wait_full = [&](int64_t q) {
    const int b = (int)(q & 1);
    mbar_wait(&bars[b], nfull[b] & 1u);
    nfull[b]++;
    tc_fence_after();
  };
  auto done_stage = [&](int64_t q) {
    const int b = (int)(q & 1);
    umma_commit(&bars[2 + b]);
    nfree[b]++;
    busy[b] = true;
  };
  auto load_feat = [&](int64_t tt, int j) {  // thread 0 only
    const int rb = j & 1;
    if (rb == 0 && pr0) { mbar_wait(&bars[4], (nring0 - 1u) & 1u); pr0 = false; }
    if (rb == 1 && pr1) { mbar_wait(&bars[5], (nring1 - 1u) & 1u); pr1 = false; }
    const uint32_t nb = (uint32_t)min(128, k0 - j * 128) * kTileM * 2;
    mbar_arrive_expect_tx(&bars[7 + rb], nb);
    img_load(s_feat + rb * 32768,
             reinterpret_cast<const uint8_t*>(a.feat_img) + (size_t)tt * kTileM * k0 * 2 + (size_t)j * 32768, nb,
             &bars[7 + rb], pol_rd);
  };
  if (t == 0 && nstages > 0) {
    issue_load(0);
    issued = 1;
  }
  bool first = true;
  for (int64_t it = 0; it < t1 - t0; ++it) {
    const int64_t tau = t1 - 1 - it;  // reverse order (see issue_load)
    const int64_t qbase = it * nst;
    TTRC(10, tau);
    // ---- stage 0: gW0^T[k][o] += F^T dz0 (features from the forward phase), gb0 += dz0^T 1
    if (t == 0 && issued < nstages) {
      issue_load(issued);
      issued++;
    }
    if (t == 0 && do_w0) {
      // feature chunks of 128 features (32 KB) from the forward phase's tile
      // image; chunks 0 and 1 of a tile were requested during the previous
      // tile's later stages (or here, for the first tile)
      if (it == 0) {
        load_feat(tau, 0);
        if (nmt > 1) load_feat(tau, 1);
      }
      for (int j = 0; j < nmt; ++j) {
        const int rb = j & 1;
        mbar_wait(&bars[7 + rb], nfeat[rb] & 1u);
        nfeat[rb]++;
        if (j == 0) wait_full(qbase);
        tc_fence_after();
        const uint32_t fb = sfe + rb * 32768;
        const uint32_t sdz = smem_addr(s_dz[qbase & 1]);
        const uint32_t idesc = idesc_f16(kTileM, W, 1, 1);
        umma_f16_run(tmem + a.col_w0 + j * W, smem_desc(fb, 128, 2048), smem_desc(sdz, 128, 2048), idesc,
                     !first ? 1u : 0u, kTileM / 16, 16, 16);
        umma_commit(&bars[4 + rb]);
        if (rb == 0) { nring0++; pr0 = true; } else { nring1++; pr1 = true; }
        if (j + 2 < nmt) load_feat(tau, j + 2);
      }
      if (!do_rest && tau > t0) {  // mode 1 has no later stages: prefetch the next tile's chunks here
        load_feat(tau - 1, 0);
        if (nmt > 1) load_feat(tau - 1, 1);
      }
    }
    if (t == 0 && !do_w0) wait_full(qbase);
    if (t == 0 && !do_rest) done_stage(qbase);
    if (t == 0 && do_rest) {
      const uint32_t sdz = smem_addr(s_dz[qbase & 1]);
      const uint32_t idesc = idesc_f16(kTileM, 16, 1, 0);
      umma_f16_run(tmem + col_b0, smem_desc(sdz, 128, 2048), smem_desc(son, 256, 128), idesc, !first ? 1u : 0u,
                   kTileM / 16, 16, 32);
      done_stage(qbase);
      TTRC(11, tau);
      // ---- stages 1..depth: gW_l^T[i][o] += [a_{l-1} | 1]^T dz_l (head: dL/dout)
      for (int l = 1; l <= depth; ++l) {
        const int64_t q = qbase + l;
        if (issued < nstages) {
          issue_load(issued);
          issued++;
        }
        wait_full(q);
        const bool head = (l == depth);
        const int b = (int)(q & 1);
        const int N = head ? 16 : W;
        const uint32_t idesc = idesc_f16(kTileM, N, 1, 1);
        const uint32_t col = head ? col_head : col_h + (l - 1) * W;
        const uint32_t sa = smem_addr(s_act[b]);
        const uint32_t bsrc = head ? smem_addr(s_dlt[b]) : smem_addr(s_dz[b]);
        umma_f16_run(tmem + col, smem_desc(sa, 128, 2048), smem_desc(bsrc, 128, 2048), idesc, !first ? 1u : 0u,
                     kTileM / 16, 16, 16);
        if (sep_bias) {
          const uint32_t cb = tmem + col_hb + (uint32_t)(l - 1) * 16u;
          if (!head) {  // gb_l[o] = dz_l^T 1: A = dz_l (outputs x samples), B = ones
            const uint32_t idb = idesc_f16(kTileM, 16, 1, 0);
            umma_f16_run(cb, smem_desc(bsrc, 128, 2048), smem_desc(son, 256, 128), idb, !first ? 1u : 0u, kTileM / 16,
                         16, 32);
          } else {  // gb_head[o] = 1^T dL/dout: A = a ones block (SBO 0: every row group reads it), B = dL/dout
            const uint32_t idb = idesc_f16(kTileM, 16, 0, 1);
            umma_f16_run(cb, smem_desc(son, 128, 0), smem_desc(bsrc, 128, 2048), idb, !first ? 1u : 0u, kTileM / 16,
                         0, 16);
          }
        }
        done_stage(q);
        if (l == 1 && tau > t0 && do_w0) {  // next tile's first feature chunks
          load_feat(tau - 1, 0);
          if (nmt > 1) load_feat(tau - 1, 1);
        }
        TTRC(11 + l, tau);
      }
    }
    first = false;
  }
  // ---- wait for every MMA, then flush per-CTA partials (zeros when no tiles)
  if (t == 0) {
    umma_commit(&bars[6]);
    mbar_wait(&bars[6], 0);
  }
  TTRC(20, 0);
  tc_fence_before();
  named_bar_sync(3, 256);
  tc_fence_after();
  float* part = a.partial + (size_t)blockIdx.x * a.P;
  const int Wr = a.width_real, K0r = 2 * a.m;
  const bool none = (t1 <= t0);
  auto rd = [&](uint32_t col, float (&v)[16]) {
    tmem_ld16(tmem + lane_off + col, v);
    tmem_ld_wait();
    if (none) {
#pragma unroll
      for (int i = 0; i < 16; ++i) v[i] = 0.f;
    }
  };
  const int64_t poff0 = a.poff[0];
  // two 16-column TMEM loads in flight per wait; streaming stores
  auto rd2 = [&](uint32_t c0, uint32_t c1, bool two, float (&v0)[16], float (&v1)[16]) {
    tmem_ld16(tmem + lane_off + c0, v0);
    if (two) tmem_ld16(tmem + lane_off + c1, v1);
    tmem_ld_wait();
    if (none) {
#pragma unroll
      for (int i = 0; i < 16; ++i) v0[i] = v1[i] = 0.f;
    }
  };
  for (int j = 0; j < (do_w0 ? nmt : 0); ++j) {
    const int k = j * 128 + row;
    float* pk = part + poff0 + k;
    for (int cc = half; cc < W / 16; cc += 4) {
      const bool two = cc + 2 < W / 16;
      float v0[16], v1[16];
      rd2(a.col_w0 + j * W + cc * 16, a.col_w0 + j * W + (cc + 2) * 16, two, v0, v1);
      if (k < K0r) {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const int o = cc * 16 + i;
          if (o < Wr) __stcs(pk + (int64_t)o * K0r, v0[i]);
        }
        if (two) {
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const int o = (cc + 2) * 16 + i;
            if (o < Wr) __stcs(pk + (int64_t)o * K0r, v1[i]);
          }
        }
      }
    }
  }
  if (do_rest && half == 0) {
    float v[16];
    rd(col_b0, v);
    if (row < Wr) part[a.poff[1] + row] = v[0];
  }
  if (do_rest && sep_bias && half == 0) {  // warps 0-3: one TMEM lane quadrant each
    for (int l = 1; l <= depth; ++l) {
      float v[16];
      rd(col_hb + (uint32_t)(l - 1) * 16u, v);
      const int64_t pb = a.poff[2 * l + 1];
      if (l < depth) {
        if (row < Wr) part[pb + row] = v[0];  // lane = output unit, column 0
      } else if (row == 0) {
        for (int o = 0; o < nd.out_dim; ++o) part[pb + o] = v[o];  // every lane holds the head's sums
      }
    }
  }
  for (int l = 1; l <= (do_rest ? depth : 0); ++l) {
    const bool head = (l == depth);
    const int N = head ? 16 : W;
    const int outs = head ? nd.out_dim : Wr;
    const uint32_t col = head ? col_head : col_h + (l - 1) * W;
    const int64_t pw = a.poff[2 * l], pb = a.poff[2 * l + 1];
    for (int cc = half; cc < N / 16; cc += 4) {
      const bool two = cc + 2 < N / 16;
      float v0[16], v1[16];
      rd2(col + cc * 16, col + (cc + 2) * 16, two, v0, v1);
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int o = cc * 16 + i;
        if (o < outs) {
          if (row < Wr) __stcs(part + pw + (int64_t)o * Wr + row, v0[i]);
          if (row == W) part[pb + o] = v0[i];  // ones column -> bias gradient
        }
        const int o1 = (cc + 2) * 16 + i;
        if (two && o1 < outs) {
          if (row < Wr) __stcs(part + pw + (int64_t)o1 * Wr + row, v1[i]);
          if (row == W) part[pb + o1] = v1[i];
        }
      }
    }
  }
  tc_fence_before();
  named_bar_sync(3, 256);
  if (t == 0)
    for (int i = 0; i < 9; ++i) mbar_inval(&bars[i]);
  TTRC(21, 0);
  if (t < 32) tmem_dealloc(tmem, 512);
}

template <bool TWO_PASS>
__global__ void __launch_bounds__(256, 1) k_train_wgrad(const WgArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  if (*a.stopped) return;
  if constexpr (TWO_PASS) {
    wg_body<1>(a, smem);
    wg_body<2>(a, smem);
  } else {
    wg_body<0>(a, smem);
  }
}

// fwd/dgrad then weight gradients of the same tiles in one launch: the
// activation / dz tile images this CTA just wrote are re-read from L2
// (same tile partition as the two-kernel form: fb_grid == wg_grid)
template <bool TWO_PASS>
__global__ void __launch_bounds__(512, 1) k_train_fbwg(const FbArgs fa, const WgArgs wa) {
  extern __shared__ __align__(1024) uint8_t smem[];
  if (*fa.stopped) return;
  fb_body(fa, smem);
  __syncthreads();
  if (threadIdx.x < 256) {
    if constexpr (TWO_PASS) {
      wg_body<1>(wa, smem);
      wg_body<2>(wa, smem);
    } else {
      wg_body<0>(wa, smem);
    }
  }
}

// ------------------------------------------------------------------ reduce + Adam
// Fixed-order sum of the per-CTA partials.  A block of 256 threads owns 32
// consecutive parameters: warp w sums partials c = w, w + 8, w + 16, ... of
// lane l's parameter (coalesced 128 B rows, ~ncta / 8 loads in two chains per
// thread instead of ncta in four), then warp 0 adds the eight warp sums as
// ((s0 + s1) + (s2 + s3)) + ((s4 + s5) + (s6 + s7)).  The order depends only
// on ncta, so every run (and the fused and data-parallel forms) is bitwise
// identical.
constexpr int kRedThreads = 256;
constexpr int kRedParams = 32;

__device__ __forceinline__ float reduce_partials32(const float* __restrict__ partial, int32_t ncta, int64_t P,
                                                   int64_t q, float* s_sum /* [8][32] */) {
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  float g0 = 0.f, g1 = 0.f;
  if (q < P) {
    int c = w;
    // eight loads in flight per thread (the sums stay in the chains' order:
    // c = w, w + 16, ... into g0 and c = w + 8, w + 24, ... into g1)
    for (; c + 56 < ncta; c += 64) {
      float v[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = partial[(size_t)(c + 8 * j) * P + q];
#pragma unroll
      for (int j = 0; j < 8; j += 2) {
        g0 += v[j];
        g1 += v[j + 1];
      }
    }
    for (; c + 8 < ncta; c += 16) {
      g0 += partial[(size_t)c * P + q];
      g1 += partial[(size_t)(c + 8) * P + q];
    }
    if (c < ncta) g0 += partial[(size_t)c * P + q];
  }
  s_sum[w * 32 + l] = g0 + g1;
  __syncthreads();
  float tot = 0.f;
  if (w == 0) {
    const float* t = s_sum + l;
    tot = ((t[0] + t[32]) + (t[64] + t[96])) + ((t[128] + t[160]) + (t[192] + t[224]));
  }
  return tot;
}

// partials -> grad[P]; per-CTA loss partials -> lossbuf[0] (data-parallel ranks all-reduce both)
__global__ void __launch_bounds__(kRedThreads) k_train_reduce(const float* __restrict__ partial, int32_t ncta,
                                                              int64_t P, float* __restrict__ grad,
                                                              const double* loss_part, int32_t nloss,
                                                              double* lossbuf, const int32_t* stopped) {
  if (*stopped) return;
  __shared__ float s_sum[8 * 32];
  const int64_t q = blockIdx.x * (int64_t)kRedParams + (threadIdx.x & 31);
  const float tot = reduce_partials32(partial, ncta, P, q, s_sum);
  if (threadIdx.x < 32 && q < P) grad[q] = tot;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    double sl = 0.0;
    for (int c = 0; c < nloss; ++c) sl += loss_part[c];
    lossbuf[0] = sl;
    // the loss rides in the gradient buffer as an f32 (hi, lo) pair, so a
    // data-parallel step all-reduces ONE buffer of P + 2 floats
    const float hi = (float)sl;
    grad[P] = hi;
    grad[P + 1] = (float)(sl - (double)hi);
  }
}

struct AdamArgs {
  const float* grad;
  const double* lossbuf;
  int64_t P;
  float* wmaster;      // [P] current params (serialized layout)
  float* mom;          // [P]
  float* vel;          // [P]
  const float* gscale; // [P] per-param gradient scale (1/size, omega, amplitude)
  const int32_t* img_off;   // [P] fp16 weight image element index or -1
  const int32_t* img_off2;  // [P] element of the transposed (dgrad) image copy or -1
  const float* img_fold;    // [P] fold factor for the image (omega [* amp])
  uint16_t* wimg;
  const int32_t* f32_dst;   // [P] index into f32 param block (bias' / head) or -1
  float* f32_block;
  const float* lr;     // [max_epochs]
  const float* c1;     // [max_epochs] float32(1 - b1^t)
  const float* c2;
  double loss_den;
  double target;
  int32_t* epoch;
  const int32_t* stopped;
  int32_t* stop_next;  // set when this epoch's pre-update loss reached the target (applied by the last block of k_train_adam)
  double* loss_hist;
  unsigned int* done_blocks;  // finished-block counter (zero between launches)
  int32_t* stopped_w;         // == stopped (written by the last block)
  int32_t* epochs_done;
  int32_t max_epochs;
  // fused single-rank form: reduce the per-CTA partials here (grad == nullptr)
  const float* partial;
  int32_t ncta;
  const double* loss_part;
  int32_t nloss;
};

// Adam on every parameter; the gradient is either the all-reduced grad[P]
// (data-parallel phase 2) or the fixed-order sum of the per-CTA partials,
// in exactly k_train_reduce's order (single rank: one launch fewer)
__global__ void __launch_bounds__(kRedThreads) k_train_adam(AdamArgs a) {
  if (*a.stopped) return;
  const int e = *a.epoch;
  const float lr = a.lr[e], c1 = a.c1[e], c2 = a.c2[e];
  __shared__ float s_sum[8 * 32];
  const int64_t q = blockIdx.x * (int64_t)kRedParams + (threadIdx.x & 31);
  // the update's per-parameter state is loaded before the reduction (its
  // latency overlaps the partial sums instead of trailing them)
  const bool upd_lane = threadIdx.x < 32 && q < a.P;
  float gs = 0.f, m0 = 0.f, v0 = 0.f, w0 = 0.f, fold = 0.f;
  int32_t io = -1, io2 = -1, fd = -1;
  if (upd_lane) {
    gs = a.gscale[q];
    m0 = a.mom[q];
    v0 = a.vel[q];
    w0 = a.wmaster[q];
    io = a.img_off[q];
    io2 = a.img_off2[q];
    fold = a.img_fold[q];
    fd = a.f32_dst[q];
  }
  float gsum = 0.f;
  if (!a.grad) gsum = reduce_partials32(a.partial, a.ncta, a.P, q, s_sum);  // block-uniform branch
  if (upd_lane) {
    if (a.grad) gsum = a.grad[q];
    const float g = gsum * gs;
    // numpy float32 arithmetic with weak python scalars (neural.py:508-523)
    float m = m0 * 0.9f;
    m = m + 0.1f * g;
    float v = v0 * 0.999f;
    v = v + 0.001f * (g * g);
    a.mom[q] = m;
    a.vel[q] = v;
    const float upd = lr * (m / c1) / (sqrtf(v / c2) + 1e-8f);
    const float w = w0 - upd;
    a.wmaster[q] = w;
    if (io >= 0) {
      __half h = __float2half_rn(w * fold);
      a.wimg[io] = *reinterpret_cast<uint16_t*>(&h);
      if (io2 >= 0) a.wimg[io2] = *reinterpret_cast<uint16_t*>(&h);
    }
    if (fd >= 0) a.f32_block[fd] = w * fold;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    double sl;
    if (a.loss_part) {
      sl = 0.0;
      for (int c = 0; c < a.nloss; ++c) sl += a.loss_part[c];
    } else {  // all-reduced (hi, lo) pair after grad[P] (k_train_reduce)
      sl = (double)a.grad[a.P] + (double)a.grad[a.P + 1];
    }
    const double loss = sl / a.loss_den;
    a.loss_hist[e] = loss;
    if (loss < a.target) *a.stop_next = 1;
  }
  // the last block to finish applies the epoch advance after every block's
  // update (the reference applies the stopping epoch's update, then breaks)
  __shared__ bool s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(a.done_blocks, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (s_last && threadIdx.x == 0) {
    __threadfence();
    *a.done_blocks = 0;
    if (*reinterpret_cast<volatile int32_t*>(a.stop_next) || e + 1 >= a.max_epochs) {
      a.stopped_w[0] = 1;
      *a.epochs_done = e + 1;
    } else {
      *a.epoch = e + 1;
      *a.epochs_done = e + 1;
    }
  }
}

#include "train_wide.cuh"

}  // namespace

// ------------------------------------------------------------------ host trainer
// CTAs that get tiles under the kernels' contiguous partition of n tiles over
// g CTAs (per = ceil(n / g)): idle CTAs would only add zero partials to the
// Adam reduction
static int busy_grid(int64_t n, int64_t g) {
  n = std::max<int64_t>(n, 1);
  const int64_t per = (n + g - 1) / g;
  return (int)((n + per - 1) / per);
}

struct nvdb_trainer {
  nvdb_train_desc d{};
  int W = 0, Wr = 0, k0 = 0, depth = 0, out_dim = 0, m = 0;
  int64_t P = 0, batch = 0, ntiles = 0, nraw = 0;
  int fb_grid = 0, wg_grid = 0, nwg = 1;
  int fb_grid0 = 0, wg_grid0 = 0, nsplit0 = 1;  // creation-time grids (buffers are sized for them)
  NetDev net{};
  uint32_t wg_smem = 0;
  SmemPlan plan{};
  std::vector<int64_t> poff;
  std::vector<std::pair<int64_t, int64_t>> layer_shape;  // (out, in)
  // device buffers
  uint8_t* blob = nullptr;   // image + bias' + head + b2pi
  float* wmaster = nullptr;
  float* mom = nullptr;
  float* vel = nullptr;
  float* gscale = nullptr;
  int32_t* img_off = nullptr;
  float* img_fold = nullptr;
  int32_t* f32_dst = nullptr;
  float* partial = nullptr;
  double* loss_part = nullptr;
  float* grad = nullptr;       // [P] summed (then all-reduced) gradient
  double* lossbuf = nullptr;   // [1] summed (then all-reduced) batch loss
  int64_t tile_begin = 0, tile_end = 0;
  uint16_t* act_img = nullptr;
  uint16_t* dz_img = nullptr;
  uint16_t* dlt_img = nullptr;
  uint16_t* feat_img = nullptr;
  int64_t* idx = nullptr;
  int32_t* idx_all = nullptr;   // [max_epochs][batch] presampled (nvdb_trainer_run / phases)
  int32_t* subset_all = nullptr;  // [nchunks][interval*batch] working subsets (sample_interval > 1)
  int32_t interval = 1, nchunks = 0, chunks_upto = 0;
  int64_t nraw_sub = 0, nraw_ep = 0;
  int32_t sampled_upto = 0;     // epochs [0, sampled_upto) are in idx_all
  int32_t host_epoch = 0;       // epochs enqueued so far
  int32_t* sflag = nullptr;
  uint32_t* sval = nullptr;
  int32_t* spos = nullptr;
  void* cub_tmp = nullptr;
  size_t cub_bytes = 0;
  unsigned long long* words = nullptr;
  float* lr = nullptr;
  float* c1 = nullptr;
  float* c2 = nullptr;
  int32_t* ctl = nullptr;  // epoch, stopped, epochs_done, stop_next, Adam done-block counter
  double* loss_hist = nullptr;
  int64_t* dpoff = nullptr;
  std::vector<std::pair<void*, size_t>> owned;  // device blocks from the block cache
  // layer-streamed path (train_wide.cuh) for nets the fused kernels cannot hold
  bool wide = false;
  LwPlan lw{};
  uint32_t nk_fwd = 0, nk_tot = 0;
  int32_t* img_off2 = nullptr;   // [P] element of the transposed (dgrad) image or -1
  uint16_t* fp_img = nullptr;    // [depth-1][ntiles][128*W] f'(z)
  LwBlock* blocks = nullptr;     // weight-gradient work blocks
  int nblocks = 0, nsplit = 1;
  int device = -1;
  cudaEvent_t done = nullptr;  // recorded after every enqueue (stream-ordered block reuse at destroy)
  bool enqueued = false;
  ~nvdb_trainer();
};

namespace {

// Device block cache for trainer buffers.  encode / encode_sequence create and
// destroy a trainer per network with the same sizes, and cudaMalloc/cudaFree
// of the ~0.3 GB per trainer (presampled indices, tile images, partials)
// cost ~90 ms per trainer; freed blocks are kept by (device, size class) and
// handed to the next trainer on the same device.  Reuse is stream ordered:
// a block returns to the cache with the event recorded after its trainer's
// last enqueued work, and is handed out only after that event completed.
// Contents are not cleared (as cudaMalloc).  nvdb_trim() releases the cache;
// a failed cudaMalloc releases it and retries once.
struct ReadyEvent {  // shared by every block of one destroyed trainer
  cudaEvent_t e = nullptr;
  ~ReadyEvent() {
    if (e) cudaEventDestroy(e);
  }
};
struct CachedBlock {
  void* p;
  std::shared_ptr<ReadyEvent> ready;  // null: no work was ever enqueued on the block
};
std::mutex g_cache_mu;
std::multimap<std::pair<int, size_t>, CachedBlock> g_cache;  // (device, size class) -> block
size_t g_cache_bytes = 0;
constexpr size_t kCacheCap = size_t(4) << 30;

size_t size_class(size_t b) {
  if (b >= (size_t(2) << 20)) return (b + (size_t(2) << 20) - 1) & ~((size_t(2) << 20) - 1);
  size_t c = 256;
  while (c < b) c <<= 1;
  return c;
}

// release every cached block (all devices); returns the bytes freed
size_t cache_release_all() {
  std::multimap<std::pair<int, size_t>, CachedBlock> drop;
  {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    drop.swap(g_cache);
    g_cache_bytes = 0;
  }
  size_t freed = 0;
  int cur = 0;
  cudaGetDevice(&cur);
  for (auto& kv : drop) {
    cudaSetDevice(kv.first.first);
    if (kv.second.ready) cudaEventSynchronize(kv.second.ready->e);
    cudaFree(kv.second.p);
    freed += kv.first.second;
  }
  cudaSetDevice(cur);
  return freed;
}

cudaError_t cached_malloc(void** p, size_t* bytes) {
  const size_t c = size_class(*bytes);
  *bytes = c;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  CachedBlock blk{nullptr, {}};
  {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    auto it = g_cache.find({dev, c});
    if (it != g_cache.end()) {
      blk = it->second;
      g_cache.erase(it);
      g_cache_bytes -= c;
    }
  }
  if (blk.p) {
    if (blk.ready) {  // the previous owner's queued kernels may still touch the block
      e = cudaEventSynchronize(blk.ready->e);
      if (e != cudaSuccess) return e;
    }
    *p = blk.p;
    return cudaSuccess;
  }
  e = cudaMalloc(p, c);
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    cache_release_all();
    e = cudaMalloc(p, c);
  }
  return e;
}

// `ready`: event after the last work that may use the block (ownership passes to the cache)
void cached_free(void* p, size_t bytes, const std::shared_ptr<ReadyEvent>& ready) {
  if (!p) return;
  int dev = 0;
  cudaGetDevice(&dev);
  {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    if (g_cache_bytes + bytes <= kCacheCap) {
      g_cache.emplace(std::make_pair(dev, bytes), CachedBlock{p, ready});
      g_cache_bytes += bytes;
      return;
    }
  }
  if (ready) cudaEventSynchronize(ready->e);
  cudaFree(p);
}

template <class T>
int dalloc(nvdb_trainer* tr, T** p, size_t count) {
  size_t bytes = sizeof(T) * std::max<size_t>(count, 1);
  void* q = nullptr;
  NVDB_CUDA_TRY(cached_malloc(&q, &bytes));
  *p = static_cast<T*>(q);
  tr->owned.emplace_back(q, bytes);
  return NVDB_OK;
}

}  // namespace

nvdb_trainer::~nvdb_trainer() {
  int cur = 0;
  cudaGetDevice(&cur);
  if (device >= 0) cudaSetDevice(device);
  // the blocks go back to the cache with the event recorded after this
  // trainer's last enqueued work (the cache now owns the event)
  std::shared_ptr<ReadyEvent> ready;
  if (done) {
    ready = std::make_shared<ReadyEvent>();
    ready->e = done;
    if (!enqueued) ready.reset();  // never recorded: nothing to wait for (destroys the event)
    done = nullptr;
  }
  for (auto& b : owned) cached_free(b.first, b.second, ready);
  owned.clear();
  cudaSetDevice(cur);
}

extern "C" int nvdb_trainer_destroy(nvdb_trainer* tr) {
  if (!tr) return NVDB_OK;
  delete tr;
  return NVDB_OK;
}

extern "C" size_t nvdb_trim(void) { return cache_release_all(); }

extern "C" int nvdb_trainer_create(const nvdb_train_desc* d, nvdb_trainer** out) {
  if (!d || !out) return fail(NVDB_EINVAL, "nvdb_trainer_create: null argument");
  const nvdb_net_desc& nd = d->net;
  if (nd.out_dim != 1 && nd.out_dim != 3) return fail(NVDB_EINVAL, "out_dim must be 1 or 3");
  if ((d->loss_kind == 1) != (nd.out_dim == 3)) return fail(NVDB_EINVAL, "ce loss needs a 3-wide head and vice versa");
  if (d->n < 1 || d->batch < 1 || d->max_epochs < 1) return fail(NVDB_EINVAL, "empty training set / batch");
  if (d->sampled && d->sample_interval > 1 && (uint64_t)d->sample_interval * (uint64_t)d->batch > 0xFFFFFFFFull)
    return fail(NVDB_EUNSUPPORTED, "sample_interval * batch >= 2^32");
  if (d->sampled && (uint64_t)d->n > 0xFFFFFFFFull) return fail(NVDB_EUNSUPPORTED, "n >= 2^32");
  std::unique_ptr<nvdb_trainer> tr(new nvdb_trainer());
  NVDB_CUDA_TRY(cudaGetDevice(&tr->device));
  NVDB_CUDA_TRY(cudaEventCreateWithFlags(&tr->done, cudaEventDisableTiming));
  tr->d = *d;
  tr->m = nd.m;
  tr->Wr = nd.width;
  tr->W = (nd.width + 15) / 16 * 16;
  tr->k0 = (2 * nd.m + kChunkK - 1) / kChunkK * kChunkK;
  tr->depth = nd.depth;
  tr->out_dim = nd.out_dim;
  const int W = tr->W, k0 = tr->k0, depth = tr->depth;
  if (W > 256 || depth > 4 || k0 > 1024) return fail(NVDB_EUNSUPPORTED, "net too large for the training kernels");
  if (d->path < 0 || d->path > 2) return fail(NVDB_EINVAL, "nvdb_train_desc.path must be 0, 1 or 2");
  // Fused narrow path (this file): weights resident in shared memory, f'(z) in
  // TMEM, weight gradients in the same launch.  The weight-gradient MMAs of
  // hidden layers and head take the activations transposed as one 128-row
  // operand (W <= 112: plus the bias' ones row; 112 < W <= 128: biases through
  // separate MMAs); fwd/dgrad keeps depth*W/2 f'(z) columns beside the W-wide
  // accumulator; wgrad keeps ceil(k0/128)*W + 16 + (depth-1)*W + 16 accumulator
  // columns (two passes when they exceed 512).  Everything else -- Table-3
  // widths, weights beyond shared memory -- takes the layer-streamed path.
  const int nmt = (k0 + 127) / 128;
  const int wg_rest = 16 + (depth - 1) * W + 16 + (W > kTileM - 16 ? depth * 16 : 0);
  const int wg_cols = nmt * W + wg_rest;
  const size_t narrow_wimg = align_up((size_t)2 * ((size_t)W * k0 + (size_t)(depth - 1) * W * W), 16);
  bool narrow_ok = W <= kTileM && !(W + depth * (W / 2) > 512 || (wg_cols > 512 && (nmt * W > 512 || wg_rest > 512)));
  if (narrow_ok) {
    const SmemPlan np_ = plan_smem((uint32_t)narrow_wimg, W, (W + depth * (W / 2) <= 256) ? 2 : 1);
    narrow_ok = np_.total <= kMaxDynSmem && kWgSmem <= kMaxDynSmem;
  }
  if (d->path == 1 && !narrow_ok)
    return fail(NVDB_EUNSUPPORTED, "net (width %d, 2m %d, depth %d) does not fit the fused narrow training kernels",
                nd.width, 2 * nd.m, depth);
  tr->wide = d->path == 2 || !narrow_ok;
  tr->nwg = (W + depth * (W / 2) <= 256) ? 2 : 1;
  tr->batch = d->sampled ? d->batch : d->n;
  tr->ntiles = (tr->batch + kTileM - 1) / kTileM;
  // ---- parameter layout (serialized: per layer W_l (out,in) then b_l)
  int64_t P = 0;
  std::vector<int> ins, outs;
  for (int l = 0; l <= depth; ++l) {
    const int in = l == 0 ? 2 * nd.m : nd.width;
    const int o = l == depth ? nd.out_dim : nd.width;
    ins.push_back(in);
    outs.push_back(o);
    tr->poff.push_back(P);
    P += (int64_t)in * o;
    tr->poff.push_back(P);
    P += o;
  }
  tr->P = P;
  // ---- image blob layout (NetDev).  Wide path: [W_0 | W_1 .. W_{d-1} | W_{d-1}^T .. W_1^T]
  tr->nk_fwd = (uint32_t)(k0 / 16 + (depth - 1) * (W / 16));
  tr->nk_tot = tr->nk_fwd + (uint32_t)((depth - 1) * (W / 16));
  const size_t wimg_bytes = tr->wide ? (size_t)tr->nk_tot * W * 32 : narrow_wimg;
  const size_t tposed_base = (size_t)W * k0 + (size_t)(depth - 1) * W * W;  // element index of W_{d-1}^T
  const size_t o_bias = align_up(wimg_bytes, 256), o_headw = align_up(o_bias + 4 * depth * W, 256);
  const size_t o_headb = align_up(o_headw + 4 * 3 * W, 256), o_b2pi = align_up(o_headb + 16, 256);
  const size_t blob_bytes = align_up(o_b2pi + 4 * 3 * (k0 / 2), 256);
  // shared-memory plan and kernel limits before any device allocation
  if (tr->wide) {
    tr->lw = plan_lw(W, depth, k0, kMaxDynSmem);
    if (tr->lw.engines < 1 || enable_max_smem(k_lw_fb) < (long long)tr->lw.total ||
        enable_max_smem(k_lw_wg) < (long long)kLwWgSmem)
      return fail(NVDB_EUNSUPPORTED, "layer-streamed training kernels exceed the shared-memory limit (%u B)",
                  tr->lw.total);
  } else if (tr->plan = plan_smem((uint32_t)wimg_bytes, W, tr->nwg), enable_max_smem(k_train_fb) < (long long)tr->plan.total ||
      enable_max_smem(k_train_wgrad<false>) < kWgSmem || enable_max_smem(k_train_wgrad<true>) < kWgSmem ||
      enable_max_smem(k_train_fbwg<false>) < (long long)std::max<uint32_t>(tr->plan.total, kWgSmem) ||
      enable_max_smem(k_train_fbwg<true>) < (long long)std::max<uint32_t>(tr->plan.total, kWgSmem))
    return fail(NVDB_EUNSUPPORTED, "training kernels exceed the shared-memory limit (%u B of resident weights "
                "and tile buffers)", tr->plan.total);
  std::vector<uint8_t> blob(blob_bytes, 0);
  std::vector<float> master(P), gscale(P), fold(P, 1.f);
  std::vector<int32_t> imgoff(P, -1), imgoff2(P, -1), f32dst(P, -1);
  const bool sine = nd.activation == NVDB_ACT_SINE;
  const float om = sine ? nd.frequency : 1.0f;
  const double inv_size = 1.0 / (double)tr->batch;
  float* f32b = reinterpret_cast<float*>(blob.data() + o_bias);  // bias' | headw | headb contiguous region
  (void)f32b;
  for (int l = 0; l <= depth; ++l) {
    const int in = ins[l], o = outs[l];
    for (int r = 0; r < o; ++r)
      for (int c = 0; c < in; ++c) {
        const int64_t q = tr->poff[2 * l] + (int64_t)r * in + c;
        master[q] = nd.weights[l][(size_t)r * in + c];
        if (l < depth) {
          const float f = (l == 0) ? om * nd.amplitude : om;
          fold[q] = f;
          gscale[q] = (float)(inv_size * f);
          const size_t e = (l == 0) ? kmajor_offset(r, c, W) / 2
                                    : ((size_t)W * k0 + (size_t)(l - 1) * W * W) + kmajor_offset(r, c, W) / 2;
          imgoff[q] = (int32_t)e;
          // the dgrad copy: (omega W_l)^T, rows = inputs c, K = outputs r; W_{d-1}^T first
          if (tr->wide && l > 0)
            imgoff2[q] = (int32_t)(tposed_base + (size_t)(depth - 1 - l) * W * W + kmajor_offset(c, r, W) / 2);
        } else {
          gscale[q] = (float)inv_size;
          fold[q] = 1.f;
          f32dst[q] = (int32_t)((o_headw - o_bias) / 4 + r * W + c);
        }
      }
    for (int r = 0; r < o; ++r) {
      const int64_t q = tr->poff[2 * l + 1] + r;
      master[q] = nd.biases[l][r];
      if (l < depth) {
        fold[q] = om;
        gscale[q] = (float)(inv_size * om);
        f32dst[q] = (int32_t)(l * W + r);
      } else {
        fold[q] = 1.f;
        gscale[q] = (float)inv_size;
        f32dst[q] = (int32_t)((o_headb - o_bias) / 4 + r);
      }
    }
  }
  // initial image and f32 params from master
  uint16_t* wimg = reinterpret_cast<uint16_t*>(blob.data());
  float* fblock = reinterpret_cast<float*>(blob.data() + o_bias);
  for (int64_t q = 0; q < P; ++q) {
    if (imgoff[q] >= 0) {
      __half h = __float2half_rn(master[q] * fold[q]);
      std::memcpy(&wimg[imgoff[q]], &h, 2);
      if (imgoff2[q] >= 0) std::memcpy(&wimg[imgoff2[q]], &h, 2);
    }
    if (f32dst[q] >= 0) fblock[f32dst[q]] = master[q] * fold[q];
  }
  float* b2 = reinterpret_cast<float*>(blob.data() + o_b2pi);
  for (int ax = 0; ax < 3; ++ax)
    for (int f = 0; f < nd.m; ++f) b2[ax * (k0 / 2) + f] = nd.b2pi[ax * nd.m + f];
  // ---- device allocations
  nvdb_trainer* t = tr.get();
  int rc = 0;
  auto chk = [&](int r) { if (r && !rc) rc = r; };
  chk(dalloc(t, &t->blob, blob_bytes));
  chk(dalloc(t, &t->wmaster, P));
  chk(dalloc(t, &t->mom, P));
  chk(dalloc(t, &t->vel, P));
  chk(dalloc(t, &t->gscale, P));
  chk(dalloc(t, &t->img_off, P));
  chk(dalloc(t, &t->img_fold, P));
  chk(dalloc(t, &t->f32_dst, P));
  chk(dalloc(t, &t->img_off2, P));
  chk(dalloc(t, &t->dpoff, t->poff.size()));
  if (rc) return rc;
  NVDB_CUDA_TRY(cudaMemcpy(t->blob, blob.data(), blob_bytes, cudaMemcpyHostToDevice));
  NVDB_CUDA_TRY(cudaMemcpy(t->wmaster, master.data(), 4 * P, cudaMemcpyHostToDevice));
  NVDB_CUDA_TRY(cudaMemset(t->mom, 0, 4 * P));
  NVDB_CUDA_TRY(cudaMemset(t->vel, 0, 4 * P));
  NVDB_CUDA_TRY(cudaMemcpy(t->gscale, gscale.data(), 4 * P, cudaMemcpyHostToDevice));
  NVDB_CUDA_TRY(cudaMemcpy(t->img_off, imgoff.data(), 4 * P, cudaMemcpyHostToDevice));
  NVDB_CUDA_TRY(cudaMemcpy(t->img_fold, fold.data(), 4 * P, cudaMemcpyHostToDevice));
  NVDB_CUDA_TRY(cudaMemcpy(t->f32_dst, f32dst.data(), 4 * P, cudaMemcpyHostToDevice));
  NVDB_CUDA_TRY(cudaMemcpy(t->img_off2, imgoff2.data(), 4 * P, cudaMemcpyHostToDevice));
  NVDB_CUDA_TRY(cudaMemcpy(t->dpoff, t->poff.data(), 8 * t->poff.size(), cudaMemcpyHostToDevice));
  NetDev& n = t->net;
  n.wimg = t->blob;
  n.bias = reinterpret_cast<const float*>(t->blob + o_bias);
  n.headw = reinterpret_cast<const float*>(t->blob + o_headw);
  n.headb = reinterpret_cast<const float*>(t->blob + o_headb);
  n.b2pi = reinterpret_cast<const float*>(t->blob + o_b2pi);
  n.wimg_bytes = (uint32_t)wimg_bytes;
  n.k0 = k0;
  n.width = W;
  n.depth = depth;
  n.out_dim = nd.out_dim;
  n.act = nd.activation;
  n.head = nd.head;
  n.expert = 0;
  // ---- per-step buffers
  const size_t tile_elems = (size_t)kTileM * W;
  {  // data-parallel share: contiguous tile range of this rank (whole batch when unsharded)
    const int64_t R = std::max(d->shard_count, 1), r = std::min<int64_t>(std::max(d->shard_rank, 0), R - 1);
    t->tile_begin = t->ntiles * r / R;
    t->tile_end = t->ntiles * (r + 1) / R;
  }
  const int64_t mine = std::max<int64_t>(t->tile_end - t->tile_begin, 1);
  t->fb_grid = (int)std::min<int64_t>(num_sms(), (mine + t->nwg - 1) / t->nwg);
  t->wg_grid = (int)std::min<int64_t>(num_sms(), mine);
  if (t->fb_grid == t->wg_grid) t->fb_grid = t->wg_grid = busy_grid(mine, t->wg_grid);
  if (t->wide) {
    t->fb_grid = (int)std::min<int64_t>(num_sms(), (mine + t->lw.engines - 1) / t->lw.engines);
    // weight-gradient blocks: every 128-row block of every layer's inputs (+ the
    // head), the bias of out-block j riding on input block j of its layer
    std::vector<LwBlock> bl;
    for (int l = 0; l <= depth; ++l) {
      const bool head = l == depth;
      const int in_pad = l == 0 ? k0 : W, in_real = l == 0 ? 2 * nd.m : nd.width;
      const int out_real = head ? nd.out_dim : nd.width;
      const int nm = (in_pad + 127) / 128;
      const int nbias = head ? 1 : (W + 127) / 128;
      for (int j = 0; j < std::max(nm, nbias); ++j) {
        LwBlock b{};
        b.layer = l;
        b.mblk = std::min(j, nm - 1);
        b.n = head ? 16 : W;
        b.bias_blk = j < nbias ? j : -1;
        b.in_real = j < nm ? in_real : 0;  // a bias-only block writes no weights
        b.out_real = out_real;
        b.a_rows = std::min(128, in_pad - b.mblk * 128);
        b.w_off = t->poff[2 * l];
        b.b_off = t->poff[2 * l + 1];
        bl.push_back(b);
      }
    }
    t->nblocks = (int)bl.size();
    t->nsplit = (int)std::max<int64_t>(1, std::min<int64_t>(mine, (num_sms() + t->nblocks - 1) / t->nblocks));
    t->wg_grid = t->nsplit;  // the Adam kernel reduces nsplit partials per parameter
    chk(dalloc(t, &t->blocks, bl.size()));
    chk(dalloc(t, &t->fp_img, (size_t)std::max(depth - 1, 1) * t->ntiles * tile_elems));
    if (rc) return rc;
    NVDB_CUDA_TRY(cudaMemcpy(t->blocks, bl.data(), sizeof(LwBlock) * bl.size(), cudaMemcpyHostToDevice));
  }
  t->fb_grid0 = t->fb_grid;
  t->wg_grid0 = t->wg_grid;
  t->nsplit0 = t->nsplit;
  chk(dalloc(t, &t->act_img, (size_t)depth * t->ntiles * tile_elems));
  chk(dalloc(t, &t->dz_img, (size_t)depth * t->ntiles * tile_elems));
  chk(dalloc(t, &t->dlt_img, (size_t)t->ntiles * kTileM * 16));
  chk(dalloc(t, &t->feat_img, (size_t)t->ntiles * kTileM * t->k0));
  chk(dalloc(t, &t->partial, (size_t)t->wg_grid * P));
  chk(dalloc(t, &t->loss_part, (size_t)t->fb_grid));
  chk(dalloc(t, &t->grad, (size_t)P + 2));  // + the loss (hi, lo) pair
  chk(dalloc(t, &t->lossbuf, 1));
  chk(dalloc(t, &t->ctl, 8));
  chk(dalloc(t, &t->loss_hist, d->max_epochs));
  chk(dalloc(t, &t->lr, d->max_epochs));
  chk(dalloc(t, &t->c1, d->max_epochs));
  chk(dalloc(t, &t->c2, d->max_epochs));
  if (rc) return rc;
  NVDB_CUDA_TRY(cudaMemset(t->ctl, 0, 32));
  NVDB_CUDA_TRY(cudaMemset(t->loss_hist, 0, 8 * d->max_epochs));
  NVDB_CUDA_TRY(cudaMemcpy(t->lr, d->lr, 4 * d->max_epochs, cudaMemcpyHostToDevice));
  NVDB_CUDA_TRY(cudaMemcpy(t->c1, d->c1, 4 * d->max_epochs, cudaMemcpyHostToDevice));
  NVDB_CUDA_TRY(cudaMemcpy(t->c2, d->c2, 4 * d->max_epochs, cudaMemcpyHostToDevice));
  if (d->sampled) {
    const uint64_t nn = (uint64_t)d->n;
    const double p_rej = nn > 1 ? (double)((uint32_t)(0u - (uint32_t)nn) % (uint32_t)nn) / 4294967296.0 : 0.0;
    t->nraw = t->batch + (int64_t)std::ceil(t->batch * p_rej * 2.0) + 1024;
    t->nraw = (t->nraw + 7) / 8 * 8;
    chk(dalloc(t, &t->idx, t->batch));
    t->interval = std::max(1, d->sample_interval);
    t->nchunks = t->interval > 1 ? (d->max_epochs + t->interval - 1) / t->interval : 0;
    if (d->n > 1) chk(dalloc(t, &t->idx_all, (size_t)d->max_epochs * t->batch));
    if (d->n > 1 && t->interval > 1) {
      chk(dalloc(t, &t->subset_all, (size_t)t->nchunks * t->interval * t->batch));
      t->nraw_sub = raw_draws((uint64_t)d->n, (int64_t)t->interval * t->batch);
      t->nraw_ep = raw_draws((uint64_t)t->interval * t->batch, t->batch);
    }
    chk(dalloc(t, &t->sflag, t->nraw));
    chk(dalloc(t, &t->sval, t->nraw));
    chk(dalloc(t, &t->spos, t->nraw));
    // words: [max_epochs][4] per-epoch draws, then (sample_interval > 1) [nchunks][4] subset draws
    chk(dalloc(t, &t->words, (size_t)4 * (d->max_epochs + t->nchunks)));
    if (rc) return rc;
    NVDB_CUDA_TRY(cudaMemcpy(t->words, d->seed_words, 32 * (size_t)(d->max_epochs + t->nchunks),
                             cudaMemcpyHostToDevice));
    cub::DeviceScan::ExclusiveSum(nullptr, t->cub_bytes, t->sflag, t->spos, (int)t->nraw);
    size_t cb = std::max<size_t>(t->cub_bytes, 16);
    void* q = nullptr;
    NVDB_CUDA_TRY(cached_malloc(&q, &cb));
    t->cub_tmp = q;
    t->owned.emplace_back(q, cb);
  }
  *out = tr.release();
  return NVDB_OK;
}

namespace {
// the completion event of the trainer's last enqueued work; not recorded while
// the stream is being captured into a graph (an event recorded in a capture
// cannot be waited on) -- the caller of graph replays orders the host itself
cudaError_t record_done(nvdb_trainer* t, cudaStream_t st) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaError_t e = cudaStreamIsCapturing(st, &cs);
  if (e != cudaSuccess) return e;
  if (cs != cudaStreamCaptureStatusNone) return cudaSuccess;
  return cudaEventRecord(t->done, st);
}

// phase 1: sampler -> fwd/dgrad -> wgrad -> partial reduction (grad, loss);
// phase 2: Adam + early stop + epoch advance.  A data-parallel caller
// all-reduces grad[P] and the loss between the two phases.
// fused_update: single rank -- the Adam kernel reduces the partials itself
int enqueue_phase(nvdb_trainer* t, int phase, cudaStream_t st, bool fused_update, int sample_ahead) {
  const nvdb_train_desc& d = t->d;
  // the device arrays (presampled indices, lr / c1 / c2, loss history) hold
  // max_epochs rows; epochs past them are refused, not run off the end
  if (t->host_epoch >= d.max_epochs)
    return fail(NVDB_EINVAL, "trainer: all %d epochs already enqueued", d.max_epochs);
  t->enqueued = true;
  int32_t* ep = t->ctl;
  int32_t* stopped = t->ctl + 1;
  if (phase == 1) {
    if (d.sampled && t->idx_all) {
      // presample this and the next epochs in one launch (one CTA per epoch)
      if (t->host_epoch >= t->sampled_upto && t->sampled_upto < d.max_epochs) {
        const int e0 = t->sampled_upto;
        const int e1 = std::min<int>(d.max_epochs, std::max(t->host_epoch, e0) + std::max(sample_ahead, 1));
        if (t->interval <= 1) {
          k_sample_epochs<<<e1 - e0, kSampThreads, 0, st>>>(t->words, (unsigned long long)d.n, t->batch, t->nraw,
                                                            e0, t->idx_all);
          NVDB_CHECK_LAUNCH();
        } else {
          // working subsets of the chunks these epochs touch, then the epochs' draws into them
          const int c1 = (e1 - 1) / t->interval + 1;
          if (c1 > t->chunks_upto) {
            const int64_t S = (int64_t)t->interval * t->batch;
            k_sample_epochs<<<c1 - t->chunks_upto, kSampThreads, 0, st>>>(
                t->words + 4 * (size_t)d.max_epochs, (unsigned long long)d.n, S, t->nraw_sub, t->chunks_upto,
                t->subset_all);
            NVDB_CHECK_LAUNCH();
            t->chunks_upto = c1;
          }
          k_sample_epochs<<<e1 - e0, kSampThreads, 0, st>>>(
              t->words, (unsigned long long)t->interval * t->batch, t->batch, t->nraw_ep, e0, t->idx_all,
              t->subset_all, (int64_t)t->interval * t->batch, t->interval);
          NVDB_CHECK_LAUNCH();
        }
        t->sampled_upto = e1;
      }
    } else if (d.sampled) {
      SampCtl c{ep, stopped, t->words, (unsigned long long)d.n, t->batch, t->nraw, t->sflag, t->sval, t->spos, t->idx};
      if (d.n == 1) {
        k_sample_ones<<<64, 256, 0, st>>>(c);
        NVDB_CHECK_LAUNCH();
      } else {
        const int64_t thr = t->nraw / 8;
        k_sample_raw<<<(int)((thr + 255) / 256), 256, 0, st>>>(c);
        NVDB_CHECK_LAUNCH();
        size_t cb = t->cub_bytes;
        NVDB_CUDA_TRY(cub::DeviceScan::ExclusiveSum(t->cub_tmp, cb, t->sflag, t->spos, (int)t->nraw, st));
        k_sample_compact<<<num_sms() * 4, 256, 0, st>>>(c);
        NVDB_CHECK_LAUNCH();
        k_sample_tail<<<1, 32, 0, st>>>(c);
        NVDB_CHECK_LAUNCH();
      }
    }
    if (t->wide) {
      LwFbArgs la{};
      la.net = t->net;
      la.nk_fwd = t->nk_fwd;
      la.nk_tot = t->nk_tot;
      la.xs = d.inputs;
      la.ys = d.targets;
      la.idx = d.sampled ? t->idx : nullptr;
      la.idx_all = (d.sampled && t->idx_all) ? t->idx_all : nullptr;
      la.epoch = ep;
      la.batch = t->batch;
      la.tile_begin = t->tile_begin;
      la.tile_end = t->tile_end;
      la.loss_kind = d.loss_kind;
      la.feat_img = t->feat_img;
      la.act_img = t->act_img;
      la.fp_img = t->fp_img;
      la.dz_img = t->dz_img;
      la.dlt_img = t->dlt_img;
      la.loss_part = t->loss_part;
      la.stopped = stopped;
      la.plan = t->lw;
      k_lw_fb<<<t->fb_grid, 128 * t->lw.engines, t->lw.total, st>>>(la);
      NVDB_CHECK_LAUNCH();
      LwWgArgs wa{};
      wa.blocks = t->blocks;
      wa.nblocks = t->nblocks;
      wa.nsplit = t->nsplit;
      wa.W = t->W;
      wa.depth = t->depth;
      wa.k0 = t->k0;
      wa.batch = t->batch;
      wa.tile_begin = t->tile_begin;
      wa.tile_end = t->tile_end;
      wa.feat_img = t->feat_img;
      wa.act_img = t->act_img;
      wa.dz_img = t->dz_img;
      wa.dlt_img = t->dlt_img;
      wa.partial = t->partial;
      wa.P = t->P;
      wa.stopped = stopped;
      k_lw_wg<<<t->nblocks * t->nsplit, 128, kLwWgSmem, st>>>(wa);
      NVDB_CHECK_LAUNCH();
      if (!fused_update) {
        k_train_reduce<<<(int)((t->P + kRedParams - 1) / kRedParams), kRedThreads, 0, st>>>(
            t->partial, t->wg_grid, t->P, t->grad, t->loss_part, t->fb_grid, t->lossbuf, stopped);
        NVDB_CHECK_LAUNCH();
      }
      NVDB_CUDA_TRY(record_done(t, st));
      return NVDB_OK;
    }
    FbArgs fa{};
    fa.idx_all = (d.sampled && t->idx_all) ? t->idx_all : nullptr;
    fa.epoch = ep;
    fa.net = t->net;
    fa.xs = d.inputs;
    fa.ys = d.targets;
    fa.idx = d.sampled ? t->idx : nullptr;
    fa.batch = t->batch;
    fa.tile_begin = t->tile_begin;
    fa.tile_end = t->tile_end;
    fa.loss_kind = d.loss_kind;
    fa.nwg = t->nwg;
    fa.act_img = t->act_img;
    fa.dz_img = t->dz_img;
    fa.dlt_img = t->dlt_img;
    fa.feat_img = t->feat_img;
    fa.loss_part = t->loss_part;
    fa.stopped = stopped;
    fa.w_off = t->plan.w_off;
    fa.region_off = t->plan.region_off;
    fa.region_bytes = t->plan.region_bytes;
    fa.small_off = t->plan.small_off;
    fa.bar_off = t->plan.bar_off;
    WgArgs wa{};
    wa.net = t->net;
    wa.m = t->m;
    wa.width_real = t->Wr;
    wa.xs = d.inputs;
    wa.idx = fa.idx;
    wa.batch = t->batch;
    wa.tile_begin = t->tile_begin;
    wa.tile_end = t->tile_end;
    wa.act_img = t->act_img;
    wa.dz_img = t->dz_img;
    wa.dlt_img = t->dlt_img;
    wa.feat_img = t->feat_img;
    wa.partial = t->partial;
    wa.P = t->P;
    wa.poff = t->dpoff;
    wa.stopped = stopped;
    const int nmt = (t->k0 + 127) / 128;
    wa.col_w0 = 0;
    wa.col_b0 = nmt * t->W;
    wa.col_h = wa.col_b0 + 16;
    wa.col_head = wa.col_h + (t->depth - 1) * t->W;
    wa.col_hb = wa.col_head + 16;
    wa.two_pass = (wa.col_hb + (t->W > kTileM - 16 ? t->depth * 16 : 0)) > 512 ? 1 : 0;
    const uint32_t fb_smem = std::max<uint32_t>(t->plan.total, 120 * 1024);
    if (t->fb_grid == t->wg_grid) {
      if (wa.two_pass)
        k_train_fbwg<true><<<t->fb_grid, 256 * t->nwg, std::max<uint32_t>(fb_smem, kWgSmem), st>>>(fa, wa);
      else
        k_train_fbwg<false><<<t->fb_grid, 256 * t->nwg, std::max<uint32_t>(fb_smem, kWgSmem), st>>>(fa, wa);
      NVDB_CHECK_LAUNCH();
    } else {
      k_train_fb<<<t->fb_grid, 256 * t->nwg, fb_smem, st>>>(fa);
      NVDB_CHECK_LAUNCH();
      if (wa.two_pass)
        k_train_wgrad<true><<<t->wg_grid, 256, kWgSmem, st>>>(wa);
      else
        k_train_wgrad<false><<<t->wg_grid, 256, kWgSmem, st>>>(wa);
      NVDB_CHECK_LAUNCH();
    }
    if (!fused_update) {
      k_train_reduce<<<(int)((t->P + kRedParams - 1) / kRedParams), kRedThreads, 0, st>>>(
          t->partial, t->wg_grid, t->P, t->grad, t->loss_part, t->fb_grid, t->lossbuf, stopped);
      NVDB_CHECK_LAUNCH();
    }
    NVDB_CUDA_TRY(record_done(t, st));
    return NVDB_OK;
  }
    AdamArgs aa{};
    aa.grad = t->grad;
    aa.lossbuf = t->lossbuf;
    aa.P = t->P;
    aa.wmaster = t->wmaster;
    aa.mom = t->mom;
    aa.vel = t->vel;
    aa.gscale = t->gscale;
    aa.img_off = t->img_off;
    aa.img_off2 = t->img_off2;
    aa.img_fold = t->img_fold;
    aa.wimg = reinterpret_cast<uint16_t*>(t->blob);
    aa.f32_dst = t->f32_dst;
    aa.f32_block = const_cast<float*>(t->net.bias);
    aa.lr = t->lr;
    aa.c1 = t->c1;
    aa.c2 = t->c2;
    aa.loss_den = (double)t->batch;
    aa.target = d.target_loss;
    aa.epoch = ep;
    aa.stopped = stopped;
    aa.stop_next = t->ctl + 3;
    if (fused_update) {
      aa.grad = nullptr;
      aa.partial = t->partial;
      aa.ncta = t->wg_grid;
      aa.loss_part = t->loss_part;
      aa.nloss = t->fb_grid;
    }
    aa.loss_hist = t->loss_hist;
    aa.done_blocks = reinterpret_cast<unsigned int*>(t->ctl + 4);
    aa.stopped_w = stopped;
    aa.epochs_done = t->ctl + 2;
    aa.max_epochs = d.max_epochs;
    k_train_adam<<<(int)((t->P + kRedParams - 1) / kRedParams), kRedThreads, 0, st>>>(aa);
    NVDB_CHECK_LAUNCH();
    ++t->host_epoch;
    NVDB_CUDA_TRY(record_done(t, st));
  return NVDB_OK;
}
}  // namespace

extern "C" int nvdb_trainer_run(nvdb_trainer* t, int32_t epochs, void* stream) {
  if (!t || epochs < 0) return fail(NVDB_EINVAL, "nvdb_trainer_run: bad args");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  for (int e = 0; e < epochs; ++e) {
    int rc = enqueue_phase(t, 1, st, true, epochs - e);
    if (!rc) rc = enqueue_phase(t, 2, st, true, 0);
    if (rc) return rc;
  }
  return NVDB_OK;
}

extern "C" int nvdb_trainer_phase(nvdb_trainer* t, int32_t phase, void* stream) {
  if (!t || (phase != 1 && phase != 2)) return fail(NVDB_EINVAL, "nvdb_trainer_phase: bad args");
  // data-parallel epochs are replayed from a captured graph: presample every
  // epoch in the first phase-1 call so later epochs launch no sampler
  return enqueue_phase(t, phase, static_cast<cudaStream_t>(stream), false, t->d.max_epochs);
}

extern "C" int nvdb_trainer_set_ctas(nvdb_trainer* t, int32_t ctas) {
  if (!t || ctas < 0) return fail(NVDB_EINVAL, "nvdb_trainer_set_ctas: bad args");
  const int c = ctas == 0 ? num_sms() : ctas;
  t->fb_grid = std::max(1, std::min(t->fb_grid0, c));
  if (t->wide) {
    t->nsplit = std::max(1, std::min(t->nsplit0, (c + t->nblocks - 1) / t->nblocks));
    t->wg_grid = t->nsplit;
  } else if (t->fb_grid0 == t->wg_grid0) {
    // the fused fwd/bwd + weight-gradient kernel keeps one tile partition
    t->fb_grid = t->wg_grid = busy_grid(t->tile_end - t->tile_begin, t->fb_grid);
  } else {
    t->wg_grid = std::max(1, std::min(t->wg_grid0, c));
  }
  return NVDB_OK;
}

extern "C" int nvdb_trainer_buffers(nvdb_trainer* t, float** grad, int64_t* nparams, double** loss) {
  if (!t || !grad || !nparams || !loss) return fail(NVDB_EINVAL, "nvdb_trainer_buffers: null argument");
  *grad = t->grad;
  *nparams = t->P;
  *loss = t->lossbuf;
  return NVDB_OK;
}

extern "C" int nvdb_trainer_packed(nvdb_trainer* t, float** buf, int64_t* nfloats) {
  if (!t || !buf || !nfloats) return fail(NVDB_EINVAL, "nvdb_trainer_packed: null argument");
  *buf = t->grad;
  *nfloats = t->P + 2;
  return NVDB_OK;
}

extern "C" int nvdb_trainer_status(const nvdb_trainer* t, int32_t* epochs_done, int32_t* stopped, double* losses,
                                   int32_t nlosses) {
  if (!t) return fail(NVDB_EINVAL, "nvdb_trainer_status: null trainer");
  // the trainer's work may be on any (non-blocking) stream: wait for the event
  // recorded after its last enqueued phase before reading its state
  if (t->enqueued) NVDB_CUDA_TRY(cudaEventSynchronize(t->done));
  int32_t ctl[3];
  NVDB_CUDA_TRY(cudaMemcpy(ctl, t->ctl, sizeof(ctl), cudaMemcpyDeviceToHost));
  if (epochs_done) *epochs_done = ctl[2];
  if (stopped) *stopped = ctl[1];
  if (losses && nlosses > 0)
    NVDB_CUDA_TRY(cudaMemcpy(losses, t->loss_hist, 8 * (size_t)std::min(nlosses, t->d.max_epochs),
                             cudaMemcpyDeviceToHost));
  return NVDB_OK;
}

// Sampler.indices(epoch) seam (encoder.py:257-267, interval == 1): the same
// kernels as the training loop, on scratch memory of its own.
// Sampler.indices(epoch) with a working subset (encoder.py:260-267):
// subset = draws(words_chunk, bound n, interval*batch), idx = subset[draws(words_epoch, bound interval*batch, batch)]
extern "C" int nvdb_sample_indices_subset(uint64_t n, int64_t batch, int32_t interval, const uint64_t* words_epoch,
                                          const uint64_t* words_chunk, int64_t* idx, void* stream) {
  if (n < 2 || batch < 1 || interval < 2 || !words_epoch || !words_chunk || !idx)
    return fail(NVDB_EINVAL, "nvdb_sample_indices_subset: bad args");
  const int64_t S = (int64_t)interval * batch;
  if (n > 0xFFFFFFFFull || S > 0xFFFFFFFFll) return fail(NVDB_EUNSUPPORTED, "bound >= 2^32");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  unsigned long long *we = nullptr, *wc = nullptr;
  int32_t *sub = nullptr, *out = nullptr;
  int rc = NVDB_OK;
  if (cudaMalloc(&we, 32) || cudaMalloc(&wc, 32) || cudaMalloc(&sub, 4 * S) || cudaMalloc(&out, 4 * batch))
    rc = fail(NVDB_ECUDA, "nvdb_sample_indices_subset: cudaMalloc");
  if (!rc) {
    cudaMemcpyAsync(we, words_epoch, 32, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(wc, words_chunk, 32, cudaMemcpyHostToDevice, st);
    k_sample_epochs<<<1, kSampThreads, 0, st>>>(wc, n, S, raw_draws(n, S), 0, sub);
    k_sample_epochs<<<1, kSampThreads, 0, st>>>(we, (unsigned long long)S, batch, raw_draws((uint64_t)S, batch), 0,
                                                out, sub, S, 1);
    k_i32_to_i64<<<(int)((batch + 255) / 256), 256, 0, st>>>(out, batch, idx);
    if (cudaStreamSynchronize(st) != cudaSuccess) rc = fail(NVDB_ECUDA, "subset sampler kernels failed");
  }
  cudaFree(we);
  cudaFree(wc);
  cudaFree(sub);
  cudaFree(out);
  return rc;
}

extern "C" int nvdb_sample_indices(uint64_t n, int64_t batch, const uint64_t* words, int64_t* idx, void* stream) {
  if (n < 1 || batch < 0 || !words || (batch > 0 && !idx)) return fail(NVDB_EINVAL, "nvdb_sample_indices: bad args");
  if (n > 0xFFFFFFFFull) return fail(NVDB_EUNSUPPORTED, "n >= 2^32");
  if (batch == 0) return NVDB_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const double p_rej = n > 1 ? (double)((uint32_t)(0u - (uint32_t)n) % (uint32_t)n) / 4294967296.0 : 0.0;
  int64_t nraw = batch + (int64_t)std::ceil(batch * p_rej * 2.0) + 1024;
  nraw = (nraw + 7) / 8 * 8;
  int32_t* ctl = nullptr;
  unsigned long long* w = nullptr;
  int32_t *flag = nullptr, *pos = nullptr;
  uint32_t* val = nullptr;
  void* tmp = nullptr;
  size_t tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, flag, pos, (int)nraw);
  int rc = NVDB_OK;
  if (cudaMalloc(&ctl, 16) || cudaMalloc(&w, 32) || cudaMalloc(&flag, 4 * nraw) || cudaMalloc(&pos, 4 * nraw) ||
      cudaMalloc(&val, 4 * nraw) || cudaMalloc(&tmp, std::max<size_t>(tb, 16)))
    rc = fail(NVDB_ECUDA, "nvdb_sample_indices: cudaMalloc");
  if (!rc) {
    cudaMemsetAsync(ctl, 0, 16, st);
    cudaMemcpyAsync(w, words, 32, cudaMemcpyHostToDevice, st);
    SampCtl c{ctl, ctl + 1, w, (unsigned long long)n, batch, nraw, flag, val, pos, idx};
    if (n == 1) {
      k_sample_ones<<<64, 256, 0, st>>>(c);
    } else {
      k_sample_raw<<<(int)((nraw / 8 + 255) / 256), 256, 0, st>>>(c);
      cub::DeviceScan::ExclusiveSum(tmp, tb, flag, pos, (int)nraw, st);
      k_sample_compact<<<num_sms() * 4, 256, 0, st>>>(c);
      k_sample_tail<<<1, 32, 0, st>>>(c);
    }
    if (cudaStreamSynchronize(st) != cudaSuccess) rc = fail(NVDB_ECUDA, "sampler kernels failed");
  }
  cudaFree(ctl);
  cudaFree(w);
  cudaFree(flag);
  cudaFree(pos);
  cudaFree(val);
  cudaFree(tmp);
  return rc;
}

extern "C" int nvdb_trainer_weights(const nvdb_trainer* t, float* const* weights, float* const* biases) {
  if (!t || !weights || !biases) return fail(NVDB_EINVAL, "nvdb_trainer_weights: null argument");
  std::vector<float> host(t->P);
  if (t->enqueued) NVDB_CUDA_TRY(cudaEventSynchronize(t->done));  // work on any stream
  NVDB_CUDA_TRY(cudaMemcpy(host.data(), t->wmaster, 4 * t->P, cudaMemcpyDeviceToHost));
  for (int l = 0; l <= t->depth; ++l) {
    const int64_t nw = t->poff[2 * l + 1] - t->poff[2 * l];
    const int64_t nb = (l < t->depth ? t->poff[2 * l + 2] : t->P) - t->poff[2 * l + 1];
    std::memcpy(weights[l], host.data() + t->poff[2 * l], 4 * nw);
    std::memcpy(biases[l], host.data() + t->poff[2 * l + 1], 4 * nb);
  }
  return NVDB_OK;
}
