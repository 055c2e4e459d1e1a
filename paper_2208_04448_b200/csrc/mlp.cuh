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
constexpr int kGroupThreads = 256;     // threads per tile group
constexpr int kCtaThreads = 512;       // two tile groups
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

// ACT: the hidden activation of every net in the launch (a container's nets
// share one TrainConfig activation), so the epilogue has no per-element branch
template <int ACT>
__global__ void __launch_bounds__(kCtaThreads, 1) mlp_eval_kernel(const MlpArgs a);

#ifdef NVDB_MLP_KERNEL_TU  // defined in exactly one translation unit (eval.cu)

// per-tile state of one group (the tile being finished and the one whose
// features are produced ahead of time)
struct TileCtx {
  int64_t first;
  int32_t count, flags;
  int64_t id;          // point id of this thread's row (outputs)
  float x0, x1, x2;    // normalised input of the row (per-point features)
  double gw;           // gate weight of the row
  bool valid, lattice;
  float lx, ly, lz;    // lattice role inputs
  uint32_t dcol;       // TMEM column of this tile's accumulator
};

template <int ACT>
__global__ void __launch_bounds__(kCtaThreads, 1) mlp_eval_kernel(const MlpArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int tid = threadIdx.x;
  const int grp = tid >> 8;              // tile group
  const int gt = tid & (kGroupThreads - 1);
  const int gw = gt >> 5;                // warp within the group
  const int quad = gw & 3;               // TMEM lane quadrant (hardware: warp id % 4)
  const int half = gw >> 2;              // which half of the pairs / columns
  const int row = quad * 32 + (gt & 31);  // tile row == TMEM lane
  const int nb = a.nbuf;                 // feature ring depth

  uint8_t* wsm = smem + a.w_off;
  float* small = reinterpret_cast<float*>(smem + a.small_off);
  float* s_bias = small + a.sm_bias;
  float* s_headw = small + a.sm_headw;
  float* s_headb = small + a.sm_headb;
  float* s_b2pi = small + a.sm_b2pi;
  float* s_lat = small + a.sm_lat;
  float* s_hx = small + a.sm_hx + grp * 128 * 4;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + a.bar_off);
  // bars[0]: weights.  Per group g at 1 + 12 g: [0..2] ring empty, [3..5] ring full
  // (256 arrivals), [6,7] layer-0 done per D region, [8] hidden layer done,
  // [9] hidden A operand full (256 arrivals)
  uint64_t* gb = bars + 1 + 12 * grp;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 32);
  __shared__ NetDev s_net;
  __shared__ ExpertDev s_exp;

  if (tid == 0) {
    mbar_init(&bars[0], 1);
    for (int g = 0; g < 2; ++g) {
      uint64_t* b = bars + 1 + 12 * g;
      for (int i = 0; i < 3; ++i) mbar_init(&b[i], 1);
      for (int i = 3; i < 6; ++i) mbar_init(&b[i], kGroupThreads);
      mbar_init(&b[6], 1);
      mbar_init(&b[7], 1);
      mbar_init(&b[8], 1);
      mbar_init(&b[9], kGroupThreads);
    }
    fence_barrier_init();
  }
  if (tid < 32) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const uint32_t tg = tmem_base + (uint32_t)(grp * 256);   // this group's TMEM columns
  const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
  const uint32_t ring_s = smem_addr(smem + a.region_off + grp * a.region_bytes);
  const uint32_t w_s = smem_addr(wsm);

  // pipeline state (parities as bit sets over the ring buffers)
  uint32_t pend = 0, epar = 0, fpar = 0;  // ring: pending commit, empty parity, full parity
  uint32_t l0par = 0, l0pend = 0;         // layer-0 done per D region
  uint32_t hpar = 0, apar = 0;            // hidden done, hidden-A full
  uint32_t cchunk = 0;                    // chunks produced by this group
  uint32_t wphase = 0;
  int loaded = -1;

  const int npairs = a.npairs_dev ? *a.npairs_dev : a.npairs;
  const int per_cta = (npairs + gridDim.x - 1) / gridDim.x;
  const int p0 = blockIdx.x * per_cta;
  const int p1 = min(npairs, p0 + per_cta);

  auto pair_net = [&](int p) { return a.tiles ? a.tiles[2 * p].net : a.implicit_net; };
  auto tile_at = [&](int p) {
    Tile t;
    if (a.tiles) {
      t = a.tiles[2 * p + grp];
    } else {
      const int64_t first = (int64_t)(2 * p + grp) * kTileM;
      t.net = a.implicit_net;
      t.first = first;
      t.flags = TF_FIRST | TF_LAST;
      t.count = (int32_t)max((int64_t)0, min((int64_t)kTileM, a.n_implicit - first));
    }
    return t;
  };

  // ---- per-tile set-up of the row inputs (decoder centres -> expert input map)
  auto setup = [&](const Tile& t, uint32_t dcol) {
    TileCtx c;
    c.first = t.first;
    c.count = t.count;
    c.flags = t.flags;
    c.dcol = dcol;
    c.valid = row < t.count;
    const int64_t pos = t.first + (c.valid ? row : 0);
    c.id = a.idx ? a.idx[pos] : pos;
    const int64_t sid = a.gather ? a.gather[c.id] : c.id;
    c.lattice = a.src_kind == SRC_LEAF_VOX && !a.idx && !a.gather && s_net.lat && t.count == kTileM &&
                (t.first & (kTileM - 1)) == 0;
    c.x0 = c.x1 = c.x2 = 0.f;
    c.gw = 1.0;
    if (!c.lattice || half == 0) {
      double cc[3];
      if (point_centre(a.src_kind, a.src, sid, cc)) {
        const double is = s_exp.inv_scale;
        c.x0 = __double2float_rn((cc[0] - s_exp.norm_origin[0]) * is);
        c.x1 = __double2float_rn((cc[1] - s_exp.norm_origin[1]) * is);
        c.x2 = __double2float_rn((cc[2] - s_exp.norm_origin[2]) * is);
        c.gw = gate_weight(s_exp.cell, a.subdomain_size, a.halo, cc);
      } else {
        const float* s = static_cast<const float*>(a.src) + 3 * sid;
        c.x0 = s[0]; c.x1 = s[1]; c.x2 = s[2];
      }
    }
    c.lx = c.ly = c.lz = 0.f;
    if (c.lattice) {
      const int lk = gt & 7, ljh = (gt >> 6) & 1, lii = gt >> 7;
      const int* o = static_cast<const int*>(a.src) + 3 * (t.first >> 9);
      const int i0 = (int)((t.first & 511) >> 6);
      const double is = s_exp.inv_scale;
      c.lx = __double2float_rn((o[0] + i0 + lii + 0.5 - s_exp.norm_origin[0]) * is);
      c.ly = __double2float_rn((o[1] + 4 * ljh + 0.5 - s_exp.norm_origin[1]) * is);
      c.lz = __double2float_rn((o[2] + lk + 0.5 - s_exp.norm_origin[2]) * is);
    }
    return c;
  };

  // ---- one feature chunk of a tile into the ring, then its layer-0 MMAs
  auto produce = [&](const TileCtx& c, int ch) {
    const int width = s_net.width, k0 = s_net.k0, mp = k0 >> 1;
    const int nch = k0 / kChunkK;
    const int b = (int)(cchunk % (uint32_t)nb);
    if ((pend >> b) & 1u) {
      mbar_wait(gb + b, ((epar >> b) & 1u) ^ 1u);
      pend &= ~(1u << b);
    }
    const uint32_t buf = ring_s + b * kChunkBytes;
    if (c.lattice) {
      // 4 pairs x 4 y-rows per thread: sincos at the first row, one rotation
      // by exp(i beta) for the second, then the Chebyshev recurrence
      // u_{j+1} = 2 cos(beta) u_j - u_{j-1} (one FFMA per cos / sin)
      const int lk = gt & 7, lpg = (gt >> 3) & 7, ljh = (gt >> 6) & 1, lii = gt >> 7;
      float cs[4][4], sn[4][4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int f = ch * (kChunkK / 2) + lpg * 4 + q;
        const float th = fmaf(c.lz, s_b2pi[2 * mp + f], fmaf(c.ly, s_b2pi[mp + f], c.lx * s_b2pi[f]));
        const float cb = s_lat[2 * f], sb = s_lat[2 * f + 1];
        __sincosf(th, &sn[q][0], &cs[q][0]);
        cs[q][1] = fmaf(cs[q][0], cb, -sn[q][0] * sb);
        sn[q][1] = fmaf(cs[q][0], sb, sn[q][0] * cb);
        const float c2 = 2.0f * cb;
        cs[q][2] = fmaf(c2, cs[q][1], -cs[q][0]);
        sn[q][2] = fmaf(c2, sn[q][1], -sn[q][0]);
        cs[q][3] = fmaf(c2, cs[q][2], -cs[q][1]);
        sn[q][3] = fmaf(c2, sn[q][2], -sn[q][1]);
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int r = lii * 64 + (4 * ljh + j) * 8 + lk;
        st_shared_v4(buf + kmajor_offset(r, lpg * 8, kTileM), pack_half2(cs[0][j], sn[0][j]),
                     pack_half2(cs[1][j], sn[1][j]), pack_half2(cs[2][j], sn[2][j]), pack_half2(cs[3][j], sn[3][j]));
      }
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint32_t h[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int f = ch * (kChunkK / 2) + half * 16 + q * 4 + j;
          const float th = fmaf(c.x2, s_b2pi[2 * mp + f], fmaf(c.x1, s_b2pi[mp + f], c.x0 * s_b2pi[f]));
          float sn, cs;
          __sincosf(th, &sn, &cs);
          h[j] = pack_half2(cs, sn);
        }
        st_shared_v4(buf + kmajor_offset(row, half * 32 + q * 8, kTileM), h[0], h[1], h[2], h[3]);
      }
    }
    fence_async_smem();
    mbar_arrive(gb + 3 + b);
    if (gt == 0) {
      mbar_wait(gb + 3 + b, (fpar >> b) & 1u);
      tc_fence_after();
      const uint32_t idesc = idesc_f16(kTileM, width, 0, 0);
#pragma unroll
      for (int s = 0; s < kChunkK / 16; ++s) {
        const uint64_t ad = smem_desc(buf + s * (2 * kTileM * 16), kTileM * 16, 128);
        const uint32_t wb = w_s + (uint32_t)(((ch * kChunkK + s * 16) >> 3) * (width >> 3) * 128);
        umma_f16(c.dcol, ad, smem_desc(wb, width * 16, 128), idesc, (ch | s) != 0);
      }
      umma_commit(gb + b);
      if (ch == nch - 1) umma_commit(gb + 6 + ((c.dcol - tg) ? 1 : 0));
    }
    fpar ^= 1u << b;
    epar ^= 1u << b;
    pend |= 1u << b;
    if (ch == nch - 1) l0pend |= 1u << ((c.dcol - tg) ? 1 : 0);
    ++cchunk;
  };

  TileCtx cur, nxt;
  bool have_nxt = false;
  for (int p = p0; p < p1; ++p) {
    if (pair_net(p) != loaded) {
      // ---- switch weights: both groups drained (no lookahead across a switch)
      __syncthreads();
      if (tid == 0) {
        s_net = a.nets[pair_net(p)];
        s_exp = a.experts[a.nets[pair_net(p)].expert];
        const NetDev& nd = a.nets[pair_net(p)];
        mbar_arrive_expect_tx(&bars[0], nd.wimg_bytes);
        for (uint32_t off = 0; off < nd.wimg_bytes; off += 32768)
          bulk_g2s(wsm + off, nd.wimg + off, min(32768u, nd.wimg_bytes - off), &bars[0]);
      }
      __syncthreads();
      {
        const NetDev& nd = s_net;
        for (int i = tid; i < nd.depth * nd.width; i += kCtaThreads) s_bias[i] = nd.bias[i];
        for (int i = tid; i < nd.out_dim * nd.width; i += kCtaThreads) s_headw[i] = nd.headw[i];
        if (tid < nd.out_dim) s_headb[tid] = nd.headb[tid];
        for (int i = tid; i < 3 * (nd.k0 / 2); i += kCtaThreads) s_b2pi[i] = nd.b2pi[i];
        if (nd.lat)
          for (int i = tid; i < nd.k0; i += kCtaThreads) s_lat[i] = nd.lat[i];
      }
      mbar_wait(&bars[0], wphase);
      wphase ^= 1u;
      __syncthreads();
      loaded = pair_net(p);
    }
    const Tile tile = tile_at(p);
    if (tile.count <= 0) continue;
    const int width = s_net.width, depth = s_net.depth, k0 = s_net.k0, out_dim = s_net.out_dim;
    const int nch = k0 / kChunkK;
    constexpr int act = ACT;
    if (!have_nxt) {
      cur = setup(tile, tg);
      for (int ch = 0; ch < nch; ++ch) produce(cur, ch);
    } else {
      cur = nxt;
    }
    have_nxt = false;
    // next tile of this group: produce its features while this tile's layers run
    bool look = false;
    if (a.two_d && p + 1 < p1 && pair_net(p + 1) == loaded) {
      const Tile t2 = tile_at(p + 1);
      if (t2.count > 0) {
        nxt = setup(t2, cur.dcol == tg ? tg + (uint32_t)width : tg);
        look = true;
      }
    }
    const int slots = depth;  // chunks of the next tile are spread over `depth` slots
    int nxt_ch = 0;
    auto produce_next = [&](int slot) {
      if (!look) return;
      const int upto = min(nch, (nch * (slot + 1)) / slots);
      for (; nxt_ch < upto; ++nxt_ch) produce(nxt, nxt_ch);
    };
    produce_next(0);
    // ---- layer 0 done for this tile
    {
      const int r = (cur.dcol - tg) ? 1 : 0;
      mbar_wait(gb + 6 + r, (l0par >> r) & 1u);
      l0par ^= 1u << r;
      l0pend &= ~(1u << r);
      tc_fence_after();
    }
    // hidden A operand (width/2 columns) after the one or two accumulator regions
    const uint32_t acol = tg + (a.two_d ? 2u : 1u) * (uint32_t)width;
    float y[kMaxOut] = {0.f, 0.f, 0.f};
    uint32_t woff = (uint32_t)(width * k0 * 2);
    for (int l = 0; l < depth; ++l) {
      const bool last = (l == depth - 1);
      const float* bl = s_bias + l * width;
      for (int cc = half; cc < width / 16; cc += 2) {
        float v[16];
        tmem_ld16(cur.dcol + lane_off + cc * 16, v);
        tmem_ld_wait();
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
              float s = y[k];
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                const float4 w4 = hw[q];
                s = fmaf(av[4 * q], w4.x, s);
                s = fmaf(av[4 * q + 1], w4.y, s);
                s = fmaf(av[4 * q + 2], w4.z, s);
                s = fmaf(av[4 * q + 3], w4.w, s);
              }
              y[k] = s;
            }
          }
        }
      }
      if (!last) {
        // hidden activations (TMEM) -> next layer: A from TMEM, B = W_{l+1} from smem
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(gb + 9);
        if (gt == 0) {
          mbar_wait(gb + 9, apar);
          tc_fence_after();
          const uint32_t idesc = idesc_f16(kTileM, width, 0, 0);
          const uint32_t wl = w_s + woff;
          for (int s = 0; s < width / 16; ++s) {
            const uint64_t bd = smem_desc(wl + (uint32_t)(s * 2 * (width >> 3) * 128), width * 16, 128);
            umma_f16_ts(cur.dcol, acol + s * 8, bd, idesc, s != 0);
          }
          umma_commit(gb + 8);
        }
        apar ^= 1u;
        woff += (uint32_t)(width * width * 2);
        produce_next(l + 1);
        mbar_wait(gb + 8, hpar);
        hpar ^= 1u;
        tc_fence_after();
      }
    }
    produce_next(slots);  // (depth == 1: nothing was interleaved)
    // head partials of the two halves of each row meet in shared memory
    if (half) {
#pragma unroll
      for (int k = 0; k < kMaxOut; ++k) s_hx[row * 4 + k] = y[k];
    }
    tc_fence_before();
    named_bar_sync(1 + grp, kGroupThreads);
    have_nxt = look;
    if (half || !cur.valid) continue;
    const int64_t id = cur.id;
    const double gwt = cur.gw;
#pragma unroll
    for (int k = 0; k < kMaxOut; ++k)
      if (k < out_dim) y[k] = (y[k] + s_hx[row * 4 + k]) + s_headb[k];

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
    bool is_first = (cur.flags & TF_FIRST) != 0, is_last = (cur.flags & TF_LAST) != 0;
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

  // ------------------------------------------------ teardown
  tc_fence_before();
  __syncthreads();
  if (tid < 32) tmem_dealloc(tmem_base, 512);
}
#endif  // NVDB_MLP_KERNEL_TU

}  // namespace nvdb
