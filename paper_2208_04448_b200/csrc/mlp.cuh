// Fused Fourier-feature MLP evaluation on tcgen05 tensor cores (sm_100a).
//
// Replaces neural.forward_block (neural.py:527-550) and the gate-blended
// evaluators around it (inference.py:39-84, partition.py:123-256): one
// persistent kernel computes, per 128-point tile,
//   centre -> expert input map (container.py:147-150, f64 then f32)
//   -> Fourier features [cos, sin] (interleaved, W0 in serialized order)
//   -> hidden layers on the tensor cores (fp16 operands, fp32 accumulate in TMEM)
//   -> head on the FMA pipe in fp32
//   -> softmax / sigmoid / identity, clamped-tent gate weight, f64 blend,
//      and the decode decision (argmax, > 0.5, clip*scale) in the epilogue.
//
// CTA = 2 tile groups of 8 warps.  A group owns one 128-point tile at a time:
// TMEM lane p (= point row p) is served by two threads (warps q and q+4 of
// the group, which share the lane quadrant), each taking half of the feature
// pairs and half of the accumulator columns; one elected thread issues the
// group's MMAs, so the tensor core runs one group's tile while the other
// group is in its MUFU/FMA epilogue.  Weights of the current net live in
// shared memory (one bulk async copy); tiles come in pairs sharing a net.
//
// Leaf-voxel tiles (a quarter of one 8^3 leaf) build their features by angle
// addition on the FMA pipe: per feature one sincos per 8 voxels along y, then
// z_{j+1} = z_j * exp(i beta_f) (beta_f = 2 pi b_fy / norm_scale), instead of
// 2m MUFU sin/cos per point.  Other sources use __sincosf per point.
#pragma once
#include <cstdint>

#include "ptx.cuh"

namespace nvdb {

constexpr int kTileM = 128;
constexpr int kChunkK = 64;            // feature K chunk (fp16 elements)
constexpr int kChunkBytes = kTileM * kChunkK * 2;   // 16 KB
constexpr int kMaxOut = 3;

enum SrcKind : int32_t {
  SRC_NORM_F32 = 0,    // already-normalised float3 inputs (forward_block seam)
  SRC_CENTER_F64 = 1,  // continuous index-space centres, double3
  SRC_COORD_I32 = 2,   // integer voxel coords, centre = c + 0.5
  SRC_LEAF_VOX = 3,    // id = leaf*512 + voxel, origins int3
  SRC_L1_SLOT = 4,     // id = node*4096 + slot, origins int3, centre = o + 8*slot + 4
};

enum OutMode : int32_t {
  OUT_RAW = 0,       // raw head outputs f32 [id][out_dim]
  OUT_PROBS = 1,     // blended f64 [id][k] + covered u8
  OUT_L1CLASS = 2,   // u8 argmax class, uncovered -> 2
  OUT_L0ACTIVE = 3,  // u8 covered & p > 0.5
  OUT_VALUE = 4,     // f32 covered ? clip?(v)*scale : background
};

enum TileFlags : int32_t { TF_FIRST = 1, TF_LAST = 2 };

enum Act : int32_t { ACT_RELU = 0, ACT_TANH = 1, ACT_SINE = 2 };
enum Head : int32_t { HEAD_LINEAR = 0, HEAD_LOGITS = 1, HEAD_BINARY = 2 };

struct alignas(16) NetDev {
  const uint8_t* wimg;  // fp16 weight image, UMMA K-major core-matrix layout
  const float* bias;    // [depth][width]  (sine: omega folded)
  const float* headw;   // [out_dim][width]
  const float* headb;   // [out_dim]
  const float* b2pi;    // [3][k0/2]
  const float* lat;     // [k0/2][2] cos/sin of the y-step angle (expert's norm scale)
  uint32_t wimg_bytes;
  int32_t k0, width, depth, out_dim, act, head, expert;
};

struct alignas(16) ExpertDev {
  double norm_origin[3];
  double norm_scale;
  double inv_scale;  // 1 / norm_scale
  int32_t cell[3];
  int32_t pad;
};

struct alignas(16) Tile {
  int32_t net;
  int32_t count;
  int32_t flags;
  int32_t pad;
  int64_t first;  // index into idx[] (or the point id itself when idx == nullptr)
};

struct MlpArgs {
  const NetDev* nets;
  const ExpertDev* experts;
  const Tile* tiles;  // nullptr -> implicit tiles: [128 i, 128 i + 128) of n_implicit points
  int32_t npairs;
  const int32_t* npairs_dev;  // non-null: pair count read on the device (built by a prior kernel)
  const uint8_t* ncand;       // non-null: per-point candidate count; first = (pass == 0),
  int32_t pass;               //           last = (ncand[id] == pass + 1); else tile flags
  int32_t implicit_net;
  int64_t n_implicit;
  int32_t src_kind;
  const int64_t* idx;     // tile position -> point id (outputs are written at [id])
  const int64_t* gather;  // point id -> source id (nullable: identity)
  const void* src;
  int32_t subdomain_size, halo;
  int32_t out_mode;
  float* out_raw;
  double* acc;  // [id][4] partial (num0..2, den) for multi-expert points
  double* out_probs;
  uint8_t* out_u8;
  float* out_f32;
  double value_scale;
  float background;
  int32_t clip;
  // shared-memory carve-up (bytes, 1024-aligned offsets)
  uint32_t w_off, region_off, region_bytes, small_off, bar_off;
  int32_t nbuf;   // feature ring buffers per group (2 or 3)
  int32_t two_d;  // 1: two accumulator regions per group (next tile's layer 0 overlaps)
  int32_t sm_bias, sm_headw, sm_headb, sm_b2pi, sm_lat, sm_hx;  // float offsets in the small region
};

// small per-net parameters staged in shared memory:
// bias [4*256] | headw [3*256] | headb [4] | b2pi [3*512] | lat [2*512] | head exchange [2][128][4]
constexpr int kSmallBias = 0;
constexpr int kSmallHeadW = 4 * 256;
constexpr int kSmallHeadB = kSmallHeadW + 3 * 256;
constexpr int kSmallB2pi = kSmallHeadB + 4;
constexpr int kSmallLat = kSmallB2pi + 3 * 512;
constexpr int kSmallHx = kSmallLat + 2 * 512;
constexpr int kSmallFloats = kSmallHx + 2 * 128 * 4;

// continuous index-space centre of point `id` of a source (decoder.py:46-47,
// 110-111, 163, 247; encoder.py:99-100).  Returns false for SRC_NORM_F32.
__device__ __forceinline__ bool point_centre(int kind, const void* src, int64_t id, double c[3]) {
  switch (kind) {
    case SRC_CENTER_F64: {
      const double* s = static_cast<const double*>(src) + 3 * id;
      c[0] = s[0]; c[1] = s[1]; c[2] = s[2];
      return true;
    }
    case SRC_COORD_I32: {
      const int* s = static_cast<const int*>(src) + 3 * id;
      c[0] = s[0] + 0.5; c[1] = s[1] + 0.5; c[2] = s[2] + 0.5;
      return true;
    }
    case SRC_LEAF_VOX: {
      const int* o = static_cast<const int*>(src) + 3 * (id >> 9);
      const int v = (int)(id & 511);
      c[0] = o[0] + (v >> 6) + 0.5; c[1] = o[1] + ((v >> 3) & 7) + 0.5; c[2] = o[2] + (v & 7) + 0.5;
      return true;
    }
    case SRC_L1_SLOT: {
      const int* o = static_cast<const int*>(src) + 3 * (id >> 12);
      const int s = (int)(id & 4095);
      c[0] = o[0] + 8.0 * (s >> 8) + 4.0; c[1] = o[1] + 8.0 * ((s >> 4) & 15) + 4.0;
      c[2] = o[2] + 8.0 * (s & 15) + 4.0;
      return true;
    }
    default:
      return false;
  }
}

// clamped-tent gate weight of the expert owning `cell` (partition.py:123-139)
__device__ __forceinline__ double gate_weight(const int cell[3], int S, int halo, const double c[3]) {
  const double h = (double)halo;
  double w = 1.0;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const double lo = (double)cell[i] * S;
    const double hi = lo + S;
    double ramp = fmin(c[i] - (lo - h), (hi + h) - c[i]) * (0.5 / h);  // exact: h is a power of two
    ramp = fmin(fmax(ramp, 0.0), 1.0);
    w *= ramp;
  }
  return w;
}

__device__ __forceinline__ float act_fn(int act, float z) {
  if (act == ACT_SINE) return __sinf(z);
  if (act == ACT_TANH) return tanhf(z);
  return fmaxf(z, 0.0f);
}

__device__ __forceinline__ void st_shared_b32(uint32_t addr, uint32_t v) {
  asm volatile("st.shared.b32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}

// Warp roles of mlp_eval_kernel: producer warps build Fourier-feature chunks
// into a shared-memory ring, one MMA warp issues every tcgen05.mma, and two
// epilogue warpgroups (one TMEM lane quadrant per warp) own alternate tiles.
constexpr int kProdWarps = 4;
constexpr int kEpiGroups = 2;
constexpr int kMmaWarp = kProdWarps + 4 * kEpiGroups;  // warp 12
constexpr int kEvalThreads = 32 * (kMmaWarp + 1);      // 416
constexpr int kMaxRing = 8;

// ACT: the hidden activation of every net in the launch (a container's nets
// share one TrainConfig activation), so the epilogue has no per-element branch
template <int ACT>
__global__ void __launch_bounds__(kEvalThreads, 1) mlp_eval_kernel(const MlpArgs a);

#ifdef NVDB_MLP_KERNEL_TU  // defined in exactly one translation unit (eval.cu)

// Pipeline (per CTA, persistent over a contiguous range of tiles):
//   producers --ring full--> MMA warp --ring empty--> producers
//   MMA warp --layer-0 done[e][r] / hidden done[e]--> epilogue group e
//   epilogue e --hidden A full[e] / region free[e][r]--> MMA warp
// The j-th non-empty tile of the CTA belongs to epilogue group j & 1; with
// `two_d` each group alternates two TMEM accumulator regions, so layer 0 of
// its next tile runs while it finishes the current one.  Hidden activations
// go back to TMEM as the fp16 A operand of the next layer (tcgen05.st).
template <int ACT>
__global__ void __launch_bounds__(kEvalThreads, 1) mlp_eval_kernel(const MlpArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int lane = tid & 31;
  const int nb = a.nbuf;

  uint8_t* wsm = smem + a.w_off;
  float* small = reinterpret_cast<float*>(smem + a.small_off);
  float* s_bias = small + a.sm_bias;
  float* s_headw = small + a.sm_headw;
  float* s_headb = small + a.sm_headb;
  float* s_b2pi = small + a.sm_b2pi;
  float* s_lat = small + a.sm_lat;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + a.bar_off);
  uint64_t* wbar = bars;            // weights landed
  uint64_t* rfull = bars + 1;       // [kMaxRing] feature chunk written (128 producer arrivals)
  uint64_t* rempty = bars + 9;      // [kMaxRing] chunk consumed (MMA commit)
  // per epilogue group e at bars + 17 + 8 e: [0,1] layer 0 done per region,
  // [2] hidden layer done, [3] hidden A written (128), [4,5] region free (128)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 40);
  __shared__ NetDev s_net;
  __shared__ ExpertDev s_exp;

  if (tid == 0) {
    mbar_init(wbar, 1);
    for (int i = 0; i < kMaxRing; ++i) {
      mbar_init(rfull + i, 32 * kProdWarps);
      mbar_init(rempty + i, 1);
    }
    for (int e = 0; e < kEpiGroups; ++e) {
      uint64_t* b = bars + 17 + 8 * e;
      mbar_init(b + 0, 1);
      mbar_init(b + 1, 1);
      mbar_init(b + 2, 1);
      mbar_init(b + 3, 128);
      mbar_init(b + 4, 128);
      mbar_init(b + 5, 128);
    }
    fence_barrier_init();
  }
  if (warp == kMmaWarp) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const uint32_t ring_s = smem_addr(smem + a.region_off);
  const uint32_t w_s = smem_addr(wsm);

  const int npairs = a.npairs_dev ? *a.npairs_dev : a.npairs;
  const int per_cta = (npairs + gridDim.x - 1) / gridDim.x;
  const int t_begin = 2 * min(npairs, (int)blockIdx.x * per_cta);
  const int t_end = 2 * min(npairs, ((int)blockIdx.x + 1) * per_cta);

  auto tile_at = [&](int t) {
    Tile tl;
    if (a.tiles) {
      tl = a.tiles[t];
    } else {
      const int64_t first = (int64_t)t * kTileM;
      tl.net = a.implicit_net;
      tl.first = first;
      tl.flags = TF_FIRST | TF_LAST;
      tl.count = (int32_t)max((int64_t)0, min((int64_t)kTileM, a.n_implicit - first));
    }
    return tl;
  };

  // ---- weight switch: every thread of the CTA, at the same tile, after all
  // work with the previous net has drained
  int loaded = -1;
  uint32_t wphase = 0;
  auto load_net = [&](int net) {
    __syncthreads();
    if (tid == 0) {
      s_net = a.nets[net];
      s_exp = a.experts[a.nets[net].expert];
      const NetDev& nd = a.nets[net];
      mbar_arrive_expect_tx(wbar, nd.wimg_bytes);
      for (uint32_t off = 0; off < nd.wimg_bytes; off += 32768)
        bulk_g2s(wsm + off, nd.wimg + off, min(32768u, nd.wimg_bytes - off), wbar);
    }
    __syncthreads();
    {
      const NetDev& nd = s_net;
      for (int i = tid; i < nd.depth * nd.width; i += kEvalThreads) s_bias[i] = nd.bias[i];
      for (int i = tid; i < nd.out_dim * nd.width; i += kEvalThreads) s_headw[i] = nd.headw[i];
      if (tid < nd.out_dim) s_headb[tid] = nd.headb[tid];
      for (int i = tid; i < 3 * (nd.k0 / 2); i += kEvalThreads) s_b2pi[i] = nd.b2pi[i];
      if (nd.lat)
        for (int i = tid; i < nd.k0; i += kEvalThreads) s_lat[i] = nd.lat[i];
    }
    mbar_wait(wbar, wphase);
    wphase ^= 1u;
    __syncthreads();
    loaded = net;
  };

  if (warp < kProdWarps) {
    // =============================================================== producers
    const int pt = tid;  // 0..127
    int slot = 0;
    uint32_t rphase = 0;
    for (int t = t_begin; t < t_end; ++t) {
      const Tile tile = tile_at(t);
      if (tile.count <= 0) continue;
      if (tile.net != loaded) load_net(tile.net);
      const int k0 = s_net.k0, mp = k0 >> 1, nch = k0 / kChunkK;
      const bool lattice = a.src_kind == SRC_LEAF_VOX && !a.idx && !a.gather && s_net.lat &&
                           tile.count == kTileM && (tile.first & (kTileM - 1)) == 0;
      const double is = s_exp.inv_scale;
      float x0 = 0.f, x1 = 0.f, x2 = 0.f;
      // lattice role: z = lk, feature quad lpg, x = lii; 8 y rows each
      const int lk = pt & 7, lpg = (pt >> 3) & 7, lii = pt >> 6;
      if (lattice) {
        const int* o = static_cast<const int*>(a.src) + 3 * (tile.first >> 9);
        const int i0 = (int)((tile.first & 511) >> 6);
        x0 = __double2float_rn((o[0] + i0 + lii + 0.5 - s_exp.norm_origin[0]) * is);
        x1 = __double2float_rn((o[1] + 0.5 - s_exp.norm_origin[1]) * is);
        x2 = __double2float_rn((o[2] + lk + 0.5 - s_exp.norm_origin[2]) * is);
      } else if (pt < tile.count) {
        const int64_t pos = tile.first + pt;
        const int64_t id = a.idx ? a.idx[pos] : pos;
        const int64_t sid = a.gather ? a.gather[id] : id;
        double cc[3];
        if (point_centre(a.src_kind, a.src, sid, cc)) {
          x0 = __double2float_rn((cc[0] - s_exp.norm_origin[0]) * is);
          x1 = __double2float_rn((cc[1] - s_exp.norm_origin[1]) * is);
          x2 = __double2float_rn((cc[2] - s_exp.norm_origin[2]) * is);
        } else {
          const float* sp = static_cast<const float*>(a.src) + 3 * sid;
          x0 = sp[0]; x1 = sp[1]; x2 = sp[2];
        }
      }
      for (int ch = 0; ch < nch; ++ch) {
        mbar_wait(rempty + slot, rphase ^ 1u);
        const uint32_t buf = ring_s + slot * kChunkBytes;
        if (lattice) {
          // 4 features x 8 y rows: one sincos, one rotation by exp(i beta),
          // then the Chebyshev recurrence u_{j+1} = 2 cos(beta) u_j - u_{j-1}
          const int f0 = ch * (kChunkK / 2) + lpg * 4;
          const float4 bx = *reinterpret_cast<const float4*>(s_b2pi + f0);
          const float4 by = *reinterpret_cast<const float4*>(s_b2pi + mp + f0);
          const float4 bz = *reinterpret_cast<const float4*>(s_b2pi + 2 * mp + f0);
          const float4 la = *reinterpret_cast<const float4*>(s_lat + 2 * f0);
          const float4 lb = *reinterpret_cast<const float4*>(s_lat + 2 * f0 + 4);
          const float bxa[4] = {bx.x, bx.y, bx.z, bx.w}, bya[4] = {by.x, by.y, by.z, by.w};
          const float bza[4] = {bz.x, bz.y, bz.z, bz.w};
          const float cba[4] = {la.x, la.z, lb.x, lb.z}, sba[4] = {la.y, la.w, lb.y, lb.w};
          float cs[4][2], sn[4][2], c2[4];
          uint32_t hp[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const float th = fmaf(x2, bza[q], fmaf(x1, bya[q], x0 * bxa[q]));
            __sincosf(th, &sn[q][0], &cs[q][0]);
            cs[q][1] = fmaf(cs[q][0], cba[q], -sn[q][0] * sba[q]);
            sn[q][1] = fmaf(cs[q][0], sba[q], sn[q][0] * cba[q]);
            c2[q] = 2.0f * cba[q];
            hp[q] = pack_half2(cs[q][0], sn[q][0]);
          }
          st_shared_v4(buf + kmajor_offset(lii * 64 + lk, lpg * 8, kTileM), hp[0], hp[1], hp[2], hp[3]);
#pragma unroll
          for (int q = 0; q < 4; ++q) hp[q] = pack_half2(cs[q][1], sn[q][1]);
          st_shared_v4(buf + kmajor_offset(lii * 64 + 8 + lk, lpg * 8, kTileM), hp[0], hp[1], hp[2], hp[3]);
#pragma unroll
          for (int jy = 2; jy < 8; ++jy) {
            const int cur = jy & 1;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              cs[q][cur] = fmaf(c2[q], cs[q][cur ^ 1], -cs[q][cur]);
              sn[q][cur] = fmaf(c2[q], sn[q][cur ^ 1], -sn[q][cur]);
              hp[q] = pack_half2(cs[q][cur], sn[q][cur]);
            }
            st_shared_v4(buf + kmajor_offset(lii * 64 + jy * 8 + lk, lpg * 8, kTileM), hp[0], hp[1], hp[2],
                         hp[3]);
          }
        } else {
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int f0 = ch * (kChunkK / 2) + q * 4;
            const float4 bx = *reinterpret_cast<const float4*>(s_b2pi + f0);
            const float4 by = *reinterpret_cast<const float4*>(s_b2pi + mp + f0);
            const float4 bz = *reinterpret_cast<const float4*>(s_b2pi + 2 * mp + f0);
            const float bxa[4] = {bx.x, bx.y, bx.z, bx.w}, bya[4] = {by.x, by.y, by.z, by.w};
            const float bza[4] = {bz.x, bz.y, bz.z, bz.w};
            uint32_t h[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const float th = fmaf(x2, bza[j], fmaf(x1, bya[j], x0 * bxa[j]));
              float sv, cv;
              __sincosf(th, &sv, &cv);
              h[j] = pack_half2(cv, sv);
            }
            st_shared_v4(buf + kmajor_offset(pt, q * 8, kTileM), h[0], h[1], h[2], h[3]);
          }
        }
        fence_async_smem();
        mbar_arrive(rfull + slot);
        if (++slot == nb) {
          slot = 0;
          rphase ^= 1u;
        }
      }
    }
  } else if (warp < kMmaWarp) {
    // =============================================================== epilogue
    const int e = (warp - kProdWarps) >> 2;
    const int quad = warp & 3;  // TMEM lane quadrant (hardware: warp id % 4)
    const int row = quad * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    uint64_t* eb = bars + 17 + 8 * e;
    const uint32_t ecol = tmem_base + (uint32_t)(e * 256);
    uint32_t l0par = 0, hpar = 0;
    int j = 0;
    constexpr int act = ACT;
    for (int t = t_begin; t < t_end; ++t) {
      const Tile tile = tile_at(t);
      if (tile.count <= 0) continue;
      if (tile.net != loaded) load_net(tile.net);
      const int mine = (j & 1) == e;
      const int jj = j >> 1;
      ++j;
      if (!mine) continue;
      const int width = s_net.width, depth = s_net.depth, out_dim = s_net.out_dim;
      const int r = a.two_d ? (jj & 1) : 0;
      const uint32_t dcol = ecol + (uint32_t)(r * width);
      const uint32_t acol = ecol + (a.two_d ? 2u : 1u) * (uint32_t)width;
      // row set-up (outputs, gate weight)
      const bool valid = row < tile.count;
      const int64_t pos = tile.first + (valid ? row : 0);
      const int64_t id = a.idx ? a.idx[pos] : pos;
      double gwt = 1.0;
      if (a.src_kind != SRC_NORM_F32) {
        const int64_t sid = a.gather ? a.gather[id] : id;
        double cc[3];
        point_centre(a.src_kind, a.src, sid, cc);
        gwt = gate_weight(s_exp.cell, a.subdomain_size, a.halo, cc);
      }
      float y[kMaxOut] = {0.f, 0.f, 0.f};
      for (int l = 0; l < depth; ++l) {
        const bool last = (l == depth - 1);
        if (l == 0) {
          mbar_wait(eb + r, (l0par >> r) & 1u);
          l0par ^= 1u << r;
        } else {
          mbar_wait(eb + 2, hpar);
          hpar ^= 1u;
        }
        tc_fence_after();
        const float* bl = s_bias + l * width;
        auto epi = [&](int cc, const float (&v)[16]) {
          float av[16];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const float4 bq = reinterpret_cast<const float4*>(bl + cc * 16)[q];
            av[4 * q + 0] = act_fn(act, v[4 * q + 0] + bq.x);
            av[4 * q + 1] = act_fn(act, v[4 * q + 1] + bq.y);
            av[4 * q + 2] = act_fn(act, v[4 * q + 2] + bq.z);
            av[4 * q + 3] = act_fn(act, v[4 * q + 3] + bq.w);
          }
          if (!last) {
            uint32_t hp[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) hp[i] = pack_half2(av[2 * i], av[2 * i + 1]);
            tmem_st8(acol + lane_off + cc * 8, hp);
          } else {
#pragma unroll
            for (int k = 0; k < kMaxOut; ++k) {
              if (k < out_dim) {
                const float4* hw = reinterpret_cast<const float4*>(s_headw + k * width + cc * 16);
                float sacc = y[k];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                  const float4 w4 = hw[q];
                  sacc = fmaf(av[4 * q], w4.x, sacc);
                  sacc = fmaf(av[4 * q + 1], w4.y, sacc);
                  sacc = fmaf(av[4 * q + 2], w4.z, sacc);
                  sacc = fmaf(av[4 * q + 3], w4.w, sacc);
                }
                y[k] = sacc;
              }
            }
          }
        };
        // up to three 16-column TMEM loads in flight per wait
        const int ncc = width / 16;
        for (int c0 = 0; c0 < ncc; c0 += 3) {
          const int m = min(3, ncc - c0);
          float v0[16], v1[16], v2[16];
          tmem_ld16(dcol + lane_off + c0 * 16, v0);
          if (m > 1) tmem_ld16(dcol + lane_off + (c0 + 1) * 16, v1);
          if (m > 2) tmem_ld16(dcol + lane_off + (c0 + 2) * 16, v2);
          tmem_ld_wait();
          epi(c0, v0);
          if (m > 1) epi(c0 + 1, v1);
          if (m > 2) epi(c0 + 2, v2);
        }
        if (!last) {
          tmem_st_wait();
          tc_fence_before();
          mbar_arrive(eb + 3);
        } else {
          tc_fence_before();
          mbar_arrive(eb + 4 + r);
        }
      }
      if (!valid) continue;
#pragma unroll
      for (int k = 0; k < kMaxOut; ++k)
        if (k < out_dim) y[k] = y[k] + s_headb[k];

      // ------------------------------------------------ output
      if (a.out_mode == OUT_RAW) {
#pragma unroll
        for (int k = 0; k < kMaxOut; ++k)
          if (k < out_dim) a.out_raw[id * out_dim + k] = y[k];
        continue;
      }
      // transform (inference.py:29-36) in float32
      float tv[kMaxOut];
      const int head = s_net.head;
      tv[1] = tv[2] = 0.f;
      if (head == HEAD_LOGITS) {  // 3-way softmax (l1 classifier heads are always 3 wide)
        const float zm = fmaxf(fmaxf(y[0], y[1]), y[2]);
        const float e0 = expf(y[0] - zm), e1 = expf(y[1] - zm), e2 = expf(y[2] - zm);
        const float ssum = (e0 + e1) + e2;
        tv[0] = e0 / ssum; tv[1] = e1 / ssum; tv[2] = e2 / ssum;
      } else if (head == HEAD_BINARY) {
        tv[0] = 1.0f / (1.0f + expf(-y[0]));
      } else {
        tv[0] = y[0];
      }
      // gate-weighted accumulation (partition.py:245-256), f64, sid order = pass order
      double num[kMaxOut], den;
      const int kk = out_dim;
#pragma unroll
      for (int k = 0; k < kMaxOut; ++k) num[k] = gwt > 0.0 ? (double)tv[k] * gwt : 0.0;
      den = gwt > 0.0 ? gwt : 0.0;
      bool is_first = (tile.flags & TF_FIRST) != 0, is_last = (tile.flags & TF_LAST) != 0;
      if (a.ncand) {
        is_first = a.pass == 0;
        is_last = (int)a.ncand[id] == a.pass + 1;
      }
      if (!is_first) {
        const double* ac = a.acc + 4 * id;
#pragma unroll
        for (int k = 0; k < kMaxOut; ++k) num[k] = ac[k] + num[k];
        den = ac[3] + den;
      }
      if (!is_last) {
        double* ac = a.acc + 4 * id;
#pragma unroll
        for (int k = 0; k < kMaxOut; ++k) ac[k] = num[k];
        ac[3] = den;
        continue;
      }
      const bool covered = den > 0.0;
      if (covered) {
#pragma unroll
        for (int k = 0; k < kMaxOut; ++k) num[k] = num[k] / den;
      }
      switch (a.out_mode) {
        case OUT_PROBS:
#pragma unroll
          for (int k = 0; k < kMaxOut; ++k)
            if (k < kk) a.out_probs[id * kk + k] = covered ? num[k] : 0.0;
          a.out_u8[id] = covered ? 1 : 0;
          break;
        case OUT_L1CLASS: {
          int best = 0;
          if (num[1] > num[best]) best = 1;
          if (num[2] > num[best]) best = 2;
          a.out_u8[id] = covered ? (uint8_t)best : (uint8_t)2;
          break;
        }
        case OUT_L0ACTIVE:
          a.out_u8[id] = (covered && num[0] > 0.5) ? 1 : 0;
          break;
        default: {  // OUT_VALUE
          double v = num[0];
          if (a.clip) v = fmin(fmax(v, -1.0), 1.0);
          a.out_f32[id] = covered ? (float)(v * a.value_scale) : a.background;
          break;
        }
      }
    }
  } else {
    // =============================================================== MMA warp
    // all lanes run the schedule; lane 0 issues.  Readiness is probed without
    // blocking so hidden-layer jobs of one group never wait behind layer 0 of
    // the other group's tile.
    const bool leader = lane == 0;
    int slot = 0;
    uint32_t rphase = 0;
    int qn[kEpiGroups] = {0, 0};            // tiles with hidden layers outstanding
    int qr[kEpiGroups][2] = {{0, 0}, {0, 0}};  // their accumulator regions (FIFO)
    int hl[kEpiGroups] = {1, 1};            // next hidden layer of the oldest one
    uint32_t apar = 0;                      // hidden-A full parity per group (bit e)
    uint32_t duse[kEpiGroups][2] = {{0, 0}, {0, 0}};  // layer-0 uses per region
    int t = t_begin, j = 0;
    bool l0_active = false;
    int ce = 0, cr = 0, ch = 0, nch = 0;
    while (true) {
      const int width = s_net.width, depth = s_net.depth;
      // ---- hidden layers (A operand from TMEM, B = W_l from shared memory)
      if (depth > 1) {
#pragma unroll
        for (int e = 0; e < kEpiGroups; ++e) {
          if (qn[e] > 0 && mbar_test(bars + 17 + 8 * e + 3, (apar >> e) & 1u)) {
            apar ^= 1u << e;
            tc_fence_after();
            const int l = hl[e];
            const uint32_t ecol = tmem_base + (uint32_t)(e * 256);
            const uint32_t dcol = ecol + (uint32_t)(qr[e][0] * width);
            const uint32_t acol = ecol + (a.two_d ? 2u : 1u) * (uint32_t)width;
            if (leader) {
              const uint32_t idesc = idesc_f16(kTileM, width, 0, 0);
              const uint32_t wl = w_s + (uint32_t)(width * s_net.k0 * 2 + (l - 1) * width * width * 2);
              for (int s = 0; s < width / 16; ++s) {
                const uint64_t bd = smem_desc(wl + (uint32_t)(s * 2 * (width >> 3) * 128), width * 16, 128);
                umma_f16_ts(dcol, acol + s * 8, bd, idesc, s != 0);
              }
              umma_commit(bars + 17 + 8 * e + 2);
            }
            __syncwarp();
            if (++hl[e] == depth) {
              hl[e] = 1;
              qr[e][0] = qr[e][1];
              --qn[e];
            }
          }
        }
      }
      // ---- layer 0 of the next tile
      if (!l0_active) {
        Tile tile;
        tile.count = 0;
        while (t < t_end) {
          tile = tile_at(t);
          if (tile.count > 0) break;
          ++t;
        }
        if (t >= t_end) {
          if (qn[0] == 0 && qn[1] == 0) break;
          continue;
        }
        if (tile.net != loaded) {
          if (qn[0] != 0 || qn[1] != 0) continue;  // drain before the weight switch
          load_net(tile.net);
          continue;
        }
        const int e = j & 1, jj = j >> 1;
        const int r = a.two_d ? (jj & 1) : 0;
        const int cap = a.two_d ? 2 : 1;
        if (depth > 1 && qn[e] >= cap) continue;
        if (duse[e][r] > 0 && !mbar_test(bars + 17 + 8 * e + 4 + r, (duse[e][r] - 1) & 1u)) continue;
        ++duse[e][r];
        l0_active = true;
        ce = e;
        cr = r;
        ch = 0;
        nch = s_net.k0 / kChunkK;
      }
      const uint32_t dcol = tmem_base + (uint32_t)(ce * 256 + cr * width);
      while (ch < nch && mbar_test(rfull + slot, rphase)) {
        tc_fence_after();
        if (leader) {
          const uint32_t buf = ring_s + slot * kChunkBytes;
          const uint32_t idesc = idesc_f16(kTileM, width, 0, 0);
#pragma unroll
          for (int s = 0; s < kChunkK / 16; ++s) {
            const uint64_t ad = smem_desc(buf + s * (2 * kTileM * 16), kTileM * 16, 128);
            const uint32_t wb = w_s + (uint32_t)(((ch * kChunkK + s * 16) >> 3) * (width >> 3) * 128);
            umma_f16(dcol, ad, smem_desc(wb, width * 16, 128), idesc, (ch | s) != 0);
          }
          umma_commit(rempty + slot);
        }
        __syncwarp();
        if (++slot == nb) {
          slot = 0;
          rphase ^= 1u;
        }
        ++ch;
      }
      if (ch == nch) {
        if (leader) umma_commit(bars + 17 + 8 * ce + cr);
        __syncwarp();
        if (depth > 1) {
          qr[ce][qn[ce]] = cr;
          ++qn[ce];
        }
        l0_active = false;
        ++j;
        ++t;
      }
    }
  }

  // ------------------------------------------------ teardown
  tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) tmem_dealloc(tmem_base, 512);
}
#endif  // NVDB_MLP_KERNEL_TU

}  // namespace nvdb
