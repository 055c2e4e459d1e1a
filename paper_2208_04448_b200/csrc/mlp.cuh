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
// CTA = up to three "tile engines" of 4 warps.  An engine owns one 128-point
// tile at a time end to end: its 128 threads build the Fourier-feature chunks
// of the tile into the engine's shared-memory slots, one elected thread issues
// the engine's tcgen05.mma for each chunk and each hidden layer, and the same
// 128 threads (TMEM lane p = point row p) run the bias/activation epilogue,
// write the fp16 activations back to TMEM as the next layer's A operand, and
// finish with the fp32 head, transform, gate and decision.  The engines share
// the net's weights in shared memory; the tensor core and MUFU are kept busy
// by whichever engines are not waiting on an MMA.
//
// Leaf-voxel tiles (a quarter of one 8^3 leaf) build their features by angle
// addition on the FMA pipe: per feature one sincos per 8 voxels along y, then
// the Chebyshev recurrence along y, instead of 2m MUFU sin/cos per point.
// Other sources use __sincosf per point.
#pragma once
#include <cstdint>
#include <type_traits>

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
  const float* bias;    // [depth][width]  (sine: omega * b)
  const float* headw;   // [out_dim][width]
  const float* headb;   // [out_dim]
  const float* b2pi;    // [3][k0/2]
  const float* lat;     // [k0/2][2] cos/sin of the y-step angle (expert's norm scale)
  uint32_t wimg_bytes;
  int32_t k0, width, depth, out_dim, act, head, expert;
  float omega;  // sine frequency, applied in fp32 in the epilogue (1 for relu / tanh)
  int32_t pad_[2];
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
  const int64_t* n_dev;       // non-null (implicit tiles): the point count is min(*n_dev, n_implicit),
                              //   read on the device (written by a prior select), no host round trip
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
  int32_t engines;  // tile engines per CTA (1..kMaxEngines); blockDim.x = 128 * engines
  int32_t tcols;    // TMEM columns per engine (the fp32 accumulator, W)
  int32_t ereg;     // shared-memory bytes per engine: 2 feature slots, reused for the hidden fp16 A tile
                    // [+ the weight ring when streaming]
  int32_t wstream;  // 1: weights do not fit in shared memory; each engine streams K = 16 weight
                    //    chunks (W x 32 bytes) through a ring of `wring` slots, wring_off into its region
  int32_t wring;     // ring slots
  uint32_t wring_off;
  uint32_t wslot_bytes;  // ring slot capacity: up to 4 consecutive K = 16 chunks (one bulk copy, one barrier round)
  int32_t wslack;        // refill up to wring - wslack slots ahead of an issuer
  int32_t sm_bias, sm_headw, sm_headb, sm_b2pi, sm_lat, sm_hx;  // float offsets in the small region
};

// small per-net parameters staged in shared memory:
// bias [4*256] | headw [3*256] | headb [4] | b2pi [3*512] | lat [8*512] | head exchange [2][128][4]
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
__device__ __forceinline__ double gate_weight(const int cell[3], int S, int halo, const double c[3],
                                              double inv2h) {  // inv2h: 0.5 / halo, hoisted by the caller
  const double h = (double)halo;
  double w = 1.0;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const double lo = (double)cell[i] * S;
    const double hi = lo + S;
    double ramp = fmin(c[i] - (lo - h), (hi + h) - c[i]) * inv2h;  // inv2h = 0.5 / h (exact: h is a power of two)
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

constexpr int kMaxEngines = 4;
constexpr int kSlots = 2;                    // feature chunk slots per engine
constexpr int kEChunkK = 48;                 // feature K per chunk (3 MMAs of K = 16)
constexpr int kEChunkBytes = kTileM * kEChunkK * 2;  // 12 KB
constexpr int kEChunkKS = 64;                // streamed weights: a feature chunk = one 4-chunk weight slot
constexpr int kEChunkBytesS = kTileM * kEChunkKS * 2;  // 16 KB
constexpr int kEvalThreads = 128 * kMaxEngines;  // largest block (512)
constexpr int kMaxWRing = 8;                 // weight ring slots per engine (streamed weights)

// ACT: the hidden activation of every net in the launch (a container's nets
// share one TrainConfig activation), so the epilogue has no per-element branch
template <int ACT>
__global__ void __launch_bounds__(kEvalThreads, 1) mlp_eval_kernel(const MlpArgs a);

#ifdef NVDB_MLP_KERNEL_TU  // defined in exactly one translation unit (eval.cu)

#ifdef NVDB_TRACE
// debug timeline of CTA 0 (trace build only): per warp a contiguous run of
// g_trace_cap records {clock64, ev << 32 | tile << 8 | warp}; no atomics
__device__ unsigned long long* g_trace = nullptr;
__device__ unsigned int g_trace_cap = 0;
__device__ unsigned int g_trace_n = 0;
#define TRC(ev, j)                                                                             \
  do {                                                                                         \
    if (blockIdx.x == 0 && g_trace && trc_n < g_trace_cap) {                                   \
      unsigned long long* _r = g_trace + 2ull * ((threadIdx.x >> 5) * g_trace_cap + trc_n++);  \
      _r[0] = clock64();                                                                       \
      _r[1] = ((unsigned long long)(ev) << 32) | ((unsigned)(j) << 8) | (unsigned)(threadIdx.x >> 5); \
    }                                                                                          \
  } while (0)
#define TRC_DECL unsigned int trc_n = 0
#else
#define TRC(ev, j) \
  do {             \
  } while (0)
#define TRC_DECL
#endif

// Per engine g (barriers at bars + 1 + 8 g): [0, kSlots) chunk slot free
// (MMA commit), [kSlots] layer done (MMA commit), [kSlots + 1] start (the
// previous engine has issued its first tile's layer 0; staggers the engines
// so one engine's feature phase overlaps another's MMA/epilogue phases).  Named barrier 1 + g syncs the
// engine's 128 threads before its elected thread issues MMAs.
template <int ACT>
__global__ void __launch_bounds__(kEvalThreads, 1) mlp_eval_kernel(const MlpArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  TRC_DECL;
  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int g = tid >> 7;    // engine
  const int p = tid & 127;   // point row = TMEM lane (engine warps are 4g..4g+3)
  const int E = a.engines;
  const int nthreads = 128 * E;

  uint8_t* wsm = smem + a.w_off;
  float* small = reinterpret_cast<float*>(smem + a.small_off);
  float* s_bias = small + a.sm_bias;
  float* s_headw = small + a.sm_headw;
  float* s_headb = small + a.sm_headb;
  float* s_b2pi = small + a.sm_b2pi;
  float* s_lat = small + a.sm_lat;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + a.bar_off);
  uint64_t* wbar = bars;                    // weights landed
  uint64_t* slot_free = bars + 1 + 8 * g;  // [kSlots]
  uint64_t* mdone = slot_free + kSlots;    // layer MMAs complete
  uint64_t* start_next = bars + 1 + 8 * (g + 1) + kSlots + 1;  // engine g+1 may start
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 33);
  uint64_t* wfull = bars + 40;                // [wring] weight chunk landed (streamed weights)
  uint64_t* wempty = wfull + kMaxWRing;      // [wring] every engine's MMA reading the chunk done
  __shared__ uint32_t s_wnext;
  __shared__ NetDev s_net;
  __shared__ ExpertDev s_exp;

  if (tid == 0) {
    mbar_init(wbar, 1);
    for (int e = 0; e < E; ++e) {
      for (int s = 0; s < kSlots + 2; ++s) mbar_init(bars + 1 + 8 * e + s, 1);

    }
    for (int s = 0; s < kMaxWRing; ++s) {
      mbar_init(bars + 40 + s, 1);
      mbar_init(bars + 40 + kMaxWRing + s, E);
    }
    s_wnext = 0;
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const uint32_t ring = smem_addr(smem + a.region_off) + (uint32_t)(g * a.ereg);
  const uint32_t w_s = smem_addr(wsm);
  const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
  const uint32_t dcol = tmem_base + (uint32_t)(g * a.tcols);
  const bool issuer = p == 0;
  // lattice feature stores (leaf-voxel tiles): row = x * 64 + y * 8 + z, with
  // z = p & 7, feature group (p >> 3) & 7, x = p >> 6; K-major core-matrix
  // offsets (kmajor_offset) without the y row (+ y * 128) and the slot base
  const uint32_t lat_row = (uint32_t)(p >> 6) * 1024u + (uint32_t)(p & 7) * 16u;
  auto lat_k = [&](uint32_t k) { return (k >> 3) * (uint32_t)(kTileM * 16) + (k & 7u) * 2u; };
  const uint32_t lat4_off = lat_row + lat_k((uint32_t)((p >> 3) & 7) * 8u);
  const uint32_t lat3_off0 = lat_row + lat_k((uint32_t)((p >> 3) & 7) * 6u);
  const uint32_t lat3_off1 = lat_row + lat_k((uint32_t)((p >> 3) & 7) * 6u + 2u);
  const uint32_t lat3_off2 = lat_row + lat_k((uint32_t)((p >> 3) & 7) * 6u + 4u);
  const double inv2h = 0.5 / (double)a.halo;

  const int64_t n_impl = a.n_dev ? min(*a.n_dev, a.n_implicit) : a.n_implicit;
  const int npairs = a.npairs_dev ? *a.npairs_dev
                     : a.n_dev ? (int)(((n_impl + kTileM - 1) / kTileM + 1) / 2) : a.npairs;
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
      tl.count = (int32_t)max((int64_t)0, min((int64_t)kTileM, n_impl - first));
    }
    return tl;
  };

  // ---- streamed weights: the net's fp16 image is a sequence of K = 16
  // chunks of W x 32 bytes (layer 0, then each hidden layer), consumed in
  // that order once per tile by every engine.  One ring of `wring` slots per
  // CTA is shared by the engines, so each chunk fetched from L2 serves all
  // engines' current tiles.  A slot holds `wp` consecutive chunks (one bulk
  // copy, one full / empty barrier round for wp MMAs: the issuing thread's
  // per-slot bookkeeping -- barrier waits, copy issue, commit -- costs
  // several MMAs' worth of clocks, tools/ubench/wstream.cu).  Slot positions
  // count up globally; any engine's issuer may claim the next position to
  // fill (s_wnext); a slot is refilled once all E engines consumed its
  // previous contents (wempty counts E).
  const int WR = a.wring;
  const uint32_t wring_s = smem_addr(smem + a.wring_off);
  uint8_t* const wring_p = smem + a.wring_off;
  uint32_t wcons = 0, wbase = 0;  // per issuer: slot position being consumed, sequence start of the net
  uint32_t wp = 1, wpc = 0;     // chunks per slot (per net), chunk within the current slot
  uint32_t wcur = 0, wph = 0;   // ring slot and barrier parity of position wcons
  uint32_t wdstep = 0;          // descriptor step of one chunk (W x 32 bytes >> 4)
  uint64_t wdesc = 0;           // B descriptor of chunk 0 of the current slot
  auto w_fill_pos = [&](uint32_t pos) {
    const uint32_t slot = pos % (uint32_t)WR;
    if (pos >= (uint32_t)WR) mbar_wait(wempty + slot, ((pos / WR) - 1) & 1u);
    const uint32_t cb = (uint32_t)s_net.width * 32u * wp;
    const uint32_t nk = s_net.wimg_bytes / cb;
    const uint32_t c = (pos - wbase) % nk;
    mbar_arrive_expect_tx(wfull + slot, cb);
    bulk_g2s(wring_p + slot * a.wslot_bytes, s_net.wimg + (size_t)c * cb, cb, wfull + slot);
  };
  auto w_refill = [&](bool blocking) {  // claim and fill positions up to WR - wslack ahead of this issuer
    while (true) {
      const uint32_t n = *reinterpret_cast<volatile uint32_t*>(&s_wnext);
      if (n >= wcons + (uint32_t)(WR - a.wslack)) break;
      if (!blocking && n >= (uint32_t)WR && !mbar_test(wempty + n % (uint32_t)WR, ((n / WR) - 1) & 1u)) break;
      if (atomicCAS(&s_wnext, n, n + 1) == n) w_fill_pos(n);
    }
  };
  // ring slot of this issuer's next position, once it landed (the slot's
  // descriptor is built here once; per chunk the issuer only adds wdstep)
  auto w_next = [&]() {
    w_refill(false);  // prefetch into slots that are already free
    while (true) {    // this issuer's own position must be claimed (blocking only for it)
      const uint32_t n = *reinterpret_cast<volatile uint32_t*>(&s_wnext);
      if (n > wcons) break;
      if (atomicCAS(&s_wnext, n, n + 1) == n) w_fill_pos(n);
    }
    mbar_wait(wfull + wcur, wph);
    wdesc = smem_desc(wring_s + wcur * a.wslot_bytes, wdstep << 3, 128);
  };
  auto w_advance = [&]() {
    ++wcons;
    if (++wcur == (uint32_t)WR) {
      wcur = 0;
      wph ^= 1u;
    }
  };
  // one K = 16 MMA with the next weight chunk of the sequence (issuer only);
  // the slot is released after its last chunk, then refilled if already free
  auto w_mma = [&](uint32_t d, uint64_t adesc, uint32_t idesc, uint32_t acc, bool ts, uint32_t a_tmem) {
    if (wpc == 0) w_next();
    const uint64_t bd = wdesc + (uint64_t)(wpc * wdstep);
    if (ts) umma_f16_ts(d, a_tmem, bd, idesc, acc);
    else umma_f16(d, adesc, bd, idesc, acc);
    if (++wpc == wp) {
      umma_commit(wempty + wcur);
      w_advance();
      wpc = 0;
      w_refill(false);
    }
  };
  // `cnt` consecutive K = 16 MMAs (A advancing 256 = 4 KB per step): whole
  // 4-chunk slots go out as one umma_f16_x4
  auto w_mma_run = [&](uint32_t d, uint64_t adesc, uint32_t idesc, uint32_t acc, int cnt) {
    for (int k = 0; k < cnt;) {
      if (wpc == 0 && wp == 4 && cnt - k >= 4) {
        w_next();
        umma_f16_x4(d, adesc, wdesc, idesc, acc, 256, wdstep);
        umma_commit(wempty + wcur);
        w_advance();
        w_refill(false);
        k += 4;
        adesc += 1024;
      } else {
        w_mma(d, adesc, idesc, acc, false, 0);
        ++k;
        adesc += 256;
      }
      acc = 1;
    }
  };
  // an engine without a tile in this (sub-)round still consumes the tile's slots
  auto w_skip_tile = [&]() {
    const uint32_t nk = s_net.wimg_bytes / ((uint32_t)s_net.width * 32u * wp);
    for (uint32_t c = 0; c < nk; ++c) {
      w_next();
      mbar_arrive(wempty + wcur);
      w_advance();
    }
  };
  // new net (all engines at the barrier, every engine consumed the same
  // positions): let the old net's prefetched chunks land, retire them for all
  // engines, restart the sequence
  auto w_restart = [&]() {
    if (tid == 0) {
      const uint32_t n = s_wnext;
      for (uint32_t pos = wcons; pos < n; ++pos) {
        const uint32_t slot = pos % (uint32_t)WR;
        mbar_wait(wfull + slot, (pos / WR) & 1u);
        for (int e = 0; e < E; ++e) mbar_arrive(wempty + slot);
      }
    }
  };

  // ---- weight switch: every thread of the CTA, at the same point of the
  // round sequence; each engine has drained its MMAs before it gets here
  int loaded = -1;
  uint32_t wphase = 0;
  auto load_net = [&](int net) {
    __syncthreads();
    if (tid == 0) {
      s_net = a.nets[net];
      s_exp = a.experts[a.nets[net].expert];
      const NetDev& nd = a.nets[net];
      if (!a.wstream) {
        mbar_arrive_expect_tx(wbar, nd.wimg_bytes);
        for (uint32_t off = 0; off < nd.wimg_bytes; off += 32768)
          bulk_g2s(wsm + off, nd.wimg + off, min(32768u, nd.wimg_bytes - off), wbar);
      }
    }
    __syncthreads();
    {
      const NetDev& nd = s_net;
      for (int i = tid; i < nd.depth * nd.width; i += nthreads) s_bias[i] = nd.bias[i];
      for (int i = tid; i < nd.out_dim * nd.width; i += nthreads) s_headw[i] = nd.headw[i];
      if (tid < nd.out_dim) s_headb[tid] = nd.headb[tid];
      for (int i = tid; i < 3 * (nd.k0 / 2); i += nthreads) s_b2pi[i] = nd.b2pi[i];
      if (nd.lat) {
        // per complex feature f: {bx, by, bz, 2 cos(beta)}, {cos(beta), sin(beta), -sin(beta), 0}
        const int mp = nd.k0 / 2;
        for (int f = tid; f < mp; f += nthreads) {
          const float cb = nd.lat[2 * f], sb = nd.lat[2 * f + 1];
          float4* L = reinterpret_cast<float4*>(s_lat) + 2 * f;
          L[0] = make_float4(nd.b2pi[f], nd.b2pi[mp + f], nd.b2pi[2 * mp + f], 2.0f * cb);
          L[1] = make_float4(cb, sb, -sb, 0.0f);
        }
      }
    }
    if (!a.wstream) {
      mbar_wait(wbar, wphase);
      wphase ^= 1u;
    } else {
      w_restart();
    }
    __syncthreads();
    if (a.wstream) {
      wcons = wbase = s_wnext;
      wpc = 0;
      wcur = wcons % (uint32_t)WR;
      wph = (wcons / (uint32_t)WR) & 1u;
      wdstep = (uint32_t)s_net.width * 2u;  // (W x 32 bytes) >> 4
      // chunks per slot: the most that fit a slot and divide every layer's chunk count
      const uint32_t pb = (uint32_t)s_net.width * 32u;
      uint32_t g = (uint32_t)s_net.k0 / 16u, h = (uint32_t)s_net.width / 16u;
      while (h) {
        const uint32_t r = g % h;
        g = h;
        h = r;
      }
      wp = 1;
      for (uint32_t q = min(a.wslot_bytes / pb, 4u); q > 1; --q)
        if (g % q == 0) {
          wp = q;
          break;
        }
    }
    loaded = net;
  };

  // stagger the engines' first tiles when the first round is uniform (all E
  // tiles non-empty, one net), so no engine can be left waiting for a start
  // signal across a weight switch
  bool stagger = false;
  if (E > 1 && t_end - t_begin >= E && !a.wstream) {  // (streamed engines pace each other through the ring)
    stagger = true;
    const Tile t0 = tile_at(t_begin);
    for (int k = 0; k < E; ++k) {
      const Tile u = tile_at(t_begin + k);
      stagger = stagger && u.count > 0 && u.net == t0.net;
    }
  }
  const bool wait_start = stagger && g > 0;

  uint32_t cc = 0;    // feature chunks this engine has written (slot = cc % kSlots)
  uint32_t mpar = 0;  // parity of the engine's next layer-done phase
  constexpr int act = ACT;

  auto process = [&](const Tile& tile, int t) {
    // feature chunk: 48 K with resident weights (two 12 KB slots beside the
    // weights), 64 K with streamed ones (one 4-chunk weight slot per feature
    // chunk; the engine region holds the wide A tile anyway)
    const int cK = a.wstream ? kEChunkKS : kEChunkK;
    const uint32_t cbytes = a.wstream ? kEChunkBytesS : kEChunkBytes;
    const int k0 = s_net.k0, mp = k0 >> 1, nch = (k0 + cK - 1) / cK;
    const int width = s_net.width, depth = s_net.depth, out_dim = s_net.out_dim;
    const uint32_t asm_ = ring;  // hidden fp16 A tile (K-major, 128 rows): the engine's slots once layer 0 is done
    const uint32_t idesc = idesc_f16(kTileM, width, 0, 0);
    const uint64_t bdesc0 = smem_desc(w_s, width * 16, 128);
    const uint32_t bstep = (uint32_t)(width >> 3) * 16u;  // (2 core-matrix columns * width/8 * 128 B) >> 4
    // lattice tiles: 128 consecutive leaf-voxel ids starting on a 128 boundary
    // (implicit tiles, or a sorted multi-expert pass whose tile kept its run)
    int64_t lfirst = tile.first;
    bool lattice = a.src_kind == SRC_LEAF_VOX && !a.gather && s_net.lat && tile.count == kTileM;
    if (lattice && a.idx) {
      lfirst = a.idx[tile.first];
      lattice = a.idx[tile.first + kTileM - 1] == lfirst + (kTileM - 1);
    }
    lattice = lattice && (lfirst & (kTileM - 1)) == 0;
    const double is = s_exp.inv_scale;
    // ------------------------------------------------ feature inputs
    float x0 = 0.f, x1 = 0.f, x2 = 0.f;
    // lattice role: z = lk, feature quad lpg, x = lii; 8 y rows each
    const int lk = p & 7, lpg = (p >> 3) & 7, lii = p >> 6;
    if (lattice) {
      const int* o = static_cast<const int*>(a.src) + 3 * (lfirst >> 9);
      const int i0 = (int)((lfirst & 511) >> 6);
      x0 = __double2float_rn((o[0] + i0 + lii + 0.5 - s_exp.norm_origin[0]) * is);
      x1 = __double2float_rn((o[1] + 0.5 - s_exp.norm_origin[1]) * is);
      x2 = __double2float_rn((o[2] + lk + 0.5 - s_exp.norm_origin[2]) * is);
    } else if (p < tile.count) {
      const int64_t pos = tile.first + p;
      const int64_t id = a.idx ? a.idx[pos] : pos;
      const int64_t sid = a.gather ? a.gather[id] : id;
      double cc3[3];
      if (point_centre(a.src_kind, a.src, sid, cc3)) {
        x0 = __double2float_rn((cc3[0] - s_exp.norm_origin[0]) * is);
        x1 = __double2float_rn((cc3[1] - s_exp.norm_origin[1]) * is);
        x2 = __double2float_rn((cc3[2] - s_exp.norm_origin[2]) * is);
      } else {
        const float* sp = static_cast<const float*>(a.src) + 3 * sid;
        x0 = sp[0]; x1 = sp[1]; x2 = sp[2];
      }
    }
    // ------------------------------------------------ layer 0: features -> MMA per chunk
    for (int ch = 0; ch < nch; ++ch, ++cc) {
      const uint32_t s = cc % kSlots;
      if (cc >= kSlots) mbar_wait(slot_free + s, ((cc / kSlots) - 1) & 1u);
      const uint32_t buf = ring + s * cbytes;
      const int kch = min(cK, k0 - ch * cK);  // K of this chunk: a multiple of 16
      const int ngrp = kch >> 3;                           // 4-feature groups in it
      if (lattice && kch == kEChunkK) {
        // 24 features x 8 z x 2 x = 384 columns of 8 y rows: three columns per
        // thread (all 128 lanes busy), one sincos + rotation per column, then
        // the Chebyshev recurrence u_{j+1} = 2 cos(beta) u_j - u_{j-1} along y
        const float4* L = reinterpret_cast<const float4*>(s_lat) + 2 * (ch * (cK / 2) + lpg * 3);
        float2 u[3][2];
        float c2[3];
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          const float4 A = L[2 * q], B = L[2 * q + 1];  // {bx, by, bz, 2 cb}, {cb, sb, -sb, 0}
          const float th = fmaf(x2, A.z, fmaf(x1, A.y, x0 * A.x));
          float s0, c0;
          __sincosf(th, &s0, &c0);
          u[q][0] = make_float2(c0, s0);
          // (c0 cb - s0 sb, c0 sb + s0 cb): the products s0 * (-sb, cb) rounded, then one fma each
          u[q][1] = __ffma2_rn(make_float2(c0, c0), make_float2(B.x, B.y), __fmul2_rn(make_float2(s0, s0), make_float2(B.z, B.x)));
          c2[q] = A.w;
        }
        const uint32_t b0 = buf + lat3_off0, b1 = buf + lat3_off1, b2 = buf + lat3_off2;
        static_for<0, 8>([&](auto jyc) {
          constexpr int jy = decltype(jyc)::value;
          if constexpr (jy >= 2) {
#pragma unroll
            for (int q = 0; q < 3; ++q)
              u[q][jy & 1] = __ffma2_rn(make_float2(c2[q], c2[q]), u[q][(jy & 1) ^ 1],
                                        make_float2(-u[q][jy & 1].x, -u[q][jy & 1].y));
          }
          st_shared_b32_at<jy * 128>(b0, pack_half2(u[0][jy & 1].x, u[0][jy & 1].y));
          st_shared_b32_at<jy * 128>(b1, pack_half2(u[1][jy & 1].x, u[1][jy & 1].y));
          st_shared_b32_at<jy * 128>(b2, pack_half2(u[2][jy & 1].x, u[2][jy & 1].y));
        });
      } else if (lattice) {
        // 4 features x 8 y rows (64-K chunks: all lanes; shorter tail chunks: lpg < ngrp)
        if (lpg < ngrp) {
        const float4* L = reinterpret_cast<const float4*>(s_lat) + 2 * (ch * (cK / 2) + lpg * 4);
        float2 u[4][2], c2[4];
        uint32_t hp[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float4 A = L[2 * q], B = L[2 * q + 1];
          const float th = fmaf(x2, A.z, fmaf(x1, A.y, x0 * A.x));
          float s0, c0;
          __sincosf(th, &s0, &c0);
          u[q][0] = make_float2(c0, s0);
          u[q][1] = __ffma2_rn(make_float2(c0, c0), make_float2(B.x, B.y), __fmul2_rn(make_float2(s0, s0), make_float2(B.z, B.x)));
          c2[q] = make_float2(A.w, A.w);
          hp[q] = pack_half2(c0, s0);
        }
        const uint32_t b4 = buf + lat4_off;
        st_shared_v4_at<0>(b4, hp[0], hp[1], hp[2], hp[3]);
#pragma unroll
        for (int q = 0; q < 4; ++q) hp[q] = pack_half2(u[q][1].x, u[q][1].y);
        st_shared_v4_at<128>(b4, hp[0], hp[1], hp[2], hp[3]);
        static_for<2, 8>([&](auto jyc) {
          constexpr int jy = decltype(jyc)::value;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            u[q][jy & 1] = __ffma2_rn(c2[q], u[q][(jy & 1) ^ 1], make_float2(-u[q][jy & 1].x, -u[q][jy & 1].y));
            hp[q] = pack_half2(u[q][jy & 1].x, u[q][jy & 1].y);
          }
          st_shared_v4_at<jy * 128>(b4, hp[0], hp[1], hp[2], hp[3]);
        });
        }
      } else {
#pragma unroll
        for (int q = 0; q < kEChunkKS / 8; ++q) {
          if (q >= ngrp) break;
          const int f0 = ch * (cK / 2) + q * 4;
          const float4 bx = *reinterpret_cast<const float4*>(s_b2pi + f0);
          const float4 by = *reinterpret_cast<const float4*>(s_b2pi + mp + f0);
          const float4 bz = *reinterpret_cast<const float4*>(s_b2pi + 2 * mp + f0);
          // theta = fma(x2, bz, fma(x1, by, x0 bx)) for two features per packed op
          // (per-lane IEEE, the scalar chain's values)
          float2 th[2];
          th[0] = __ffma2_rn(make_float2(x2, x2), make_float2(bz.x, bz.y),
                             __ffma2_rn(make_float2(x1, x1), make_float2(by.x, by.y),
                                        __fmul2_rn(make_float2(x0, x0), make_float2(bx.x, bx.y))));
          th[1] = __ffma2_rn(make_float2(x2, x2), make_float2(bz.z, bz.w),
                             __ffma2_rn(make_float2(x1, x1), make_float2(by.z, by.w),
                                        __fmul2_rn(make_float2(x0, x0), make_float2(bx.z, bx.w))));
          uint32_t h[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            float sv, cv;
            __sincosf((j & 1) ? th[j >> 1].y : th[j >> 1].x, &sv, &cv);
            h[j] = pack_half2(cv, sv);
          }
          st_shared_v4(buf + kmajor_offset(p, q * 8, kTileM), h[0], h[1], h[2], h[3]);
        }
      }
      fence_async_smem();
      named_bar_sync(1 + g, 128);
      if (!a.wstream && kch == 48) {
        // resident weights: the engine's first warp issues converged (elected lane)
        if ((warp & 3) == 0) {
          tc_fence_after();
          umma_f16_x3_w(dcol, smem_desc(buf, kTileM * 16, 128),
                        bdesc0 + (uint64_t)(ch * (kEChunkK / 16) * bstep), idesc, ch != 0, 256, bstep);
          umma_commit_w(slot_free + s);
          if (ch == nch - 1) umma_commit_w(mdone);
        }
      } else if (issuer) {
        tc_fence_after();
        // descriptors: start-address field += byte offset >> 4 (no carry: smem < 256 KB);
        // one K = 16 step = 2 core-matrix columns of the operand
        const uint64_t ad = smem_desc(buf, kTileM * 16, 128);
        if (a.wstream) {
          w_mma_run(dcol, ad, idesc, ch != 0 ? 1u : 0u, kch >> 4);
        } else {
          const uint64_t bd = bdesc0 + (uint64_t)(ch * (kEChunkK / 16) * bstep);
          if (kch == 48) {  // one asm block (one ELECT / R2UR sequence) for the chunk's 3 MMAs
            umma_f16_x3(dcol, ad, bd, idesc, ch != 0, 256, bstep);
          } else {
            umma_f16(dcol, ad, bd, idesc, ch != 0);
            if (kch > 16) umma_f16(dcol, ad + 256, bd + bstep, idesc, 1);
            if (kch > 32) umma_f16(dcol, ad + 512, bd + 2 * bstep, idesc, 1);
          }
        }
        umma_commit(slot_free + s);
        if (ch == nch - 1) umma_commit(mdone);
      }
    }
    if (stagger) {
      stagger = false;
      if (issuer && g + 1 < E) mbar_arrive(start_next);
    }
    if (issuer) TRC(1, t);
    // ------------------------------------------------ hidden layers + head
    float y[kMaxOut] = {0.f, 0.f, 0.f};
    for (int l = 0; l < depth; ++l) {
      const bool last = (l == depth - 1);
      mbar_wait(mdone, mpar);
      mpar ^= 1u;
      tc_fence_after();
      if (issuer) TRC(2 + l, t);
      const float* bl = s_bias + l * width;
      const float om = s_net.omega;
      // batches of NB 16-column TMEM loads, then straight-line bias /
      // activation / pack (no branches inside a batch, so the MUFU ops of one
      // group overlap the packing and stores of the previous one)
      auto batch = [&](auto nb_c, auto last_c, int c0) {
        constexpr int NB = decltype(nb_c)::value;
        constexpr bool LAST = decltype(last_c)::value;
        float v[NB][16];
#pragma unroll
        for (int b = 0; b < NB; ++b) tmem_ld16(dcol + lane_off + (c0 + b) * 16, v[b]);
        tmem_ld_wait();
#pragma unroll
        for (int b = 0; b < NB; ++b) {
          float av[16];
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4) {
            // sin(omega (W a + b)) = sin(fma(acc, omega, omega b)): the fp16
            // weights stay unscaled (exact for 16-bit containers), omega in fp32
            const float4 bq = reinterpret_cast<const float4*>(bl + (c0 + b) * 16)[q4];
            if constexpr (ACT == ACT_SINE) {
              const float2 om2 = make_float2(om, om);
              const float2 z01 = __ffma2_rn(make_float2(v[b][4 * q4 + 0], v[b][4 * q4 + 1]), om2,
                                            make_float2(bq.x, bq.y));
              const float2 z23 = __ffma2_rn(make_float2(v[b][4 * q4 + 2], v[b][4 * q4 + 3]), om2,
                                            make_float2(bq.z, bq.w));
              av[4 * q4 + 0] = act_fn(act, z01.x);
              av[4 * q4 + 1] = act_fn(act, z01.y);
              av[4 * q4 + 2] = act_fn(act, z23.x);
              av[4 * q4 + 3] = act_fn(act, z23.y);
            } else {
              av[4 * q4 + 0] = act_fn(act, v[b][4 * q4 + 0] + bq.x);
              av[4 * q4 + 1] = act_fn(act, v[b][4 * q4 + 1] + bq.y);
              av[4 * q4 + 2] = act_fn(act, v[b][4 * q4 + 2] + bq.z);
              av[4 * q4 + 3] = act_fn(act, v[b][4 * q4 + 3] + bq.w);
            }
          }
          if constexpr (!LAST) {
            uint32_t hp[8];
#pragma unroll
            for (int i2 = 0; i2 < 8; ++i2) hp[i2] = pack_half2(av[2 * i2], av[2 * i2 + 1]);
            const uint32_t ao = asm_ + kmajor_offset(p, (c0 + b) * 16, kTileM);
            st_shared_v4(ao, hp[0], hp[1], hp[2], hp[3]);
            st_shared_v4(ao + kTileM * 16, hp[4], hp[5], hp[6], hp[7]);  // next 8-column core-matrix column
          } else {
#pragma unroll
            for (int k = 0; k < kMaxOut; ++k) {
              if (k < out_dim) {
                const float4* hw = reinterpret_cast<const float4*>(s_headw + k * width + (c0 + b) * 16);
                // four short partial sums as two fp32x2 chains (even / odd columns)
                float2 sp[2];
#pragma unroll
                for (int h2 = 0; h2 < 2; ++h2) {
                  const float4 wa = hw[2 * h2], wb = hw[2 * h2 + 1];
                  const float* a8 = av + 8 * h2;
                  sp[h2] = __fmul2_rn(make_float2(a8[0], a8[1]), make_float2(wa.x, wa.y));
                  sp[h2] = __ffma2_rn(make_float2(a8[2], a8[3]), make_float2(wa.z, wa.w), sp[h2]);
                  sp[h2] = __ffma2_rn(make_float2(a8[4], a8[5]), make_float2(wb.x, wb.y), sp[h2]);
                  sp[h2] = __ffma2_rn(make_float2(a8[6], a8[7]), make_float2(wb.z, wb.w), sp[h2]);
                }
                y[k] += (sp[0].x + sp[0].y) + (sp[1].x + sp[1].y);
              }
            }
          }
        }
      };
      const int ncc = width / 16;
      auto run_layer = [&](auto last_c) {
        int c0 = 0;
        for (; c0 + 2 <= ncc; c0 += 2) batch(std::integral_constant<int, 2>{}, last_c, c0);
        for (; c0 < ncc; ++c0) batch(std::integral_constant<int, 1>{}, last_c, c0);
      };
      if (last) run_layer(std::true_type{});
      else run_layer(std::false_type{});
      tc_fence_before();
      if (!last && !a.wstream && (width % 48) == 0) {
        // resident weights, W a multiple of 48: the layer's MMAs in threes from
        // the engine's first warp, converged (as the feature chunks)
        fence_async_smem();
        tc_fence_before();
        named_bar_sync(1 + g, 128);
        if ((warp & 3) == 0) {
          tc_fence_after();
          uint64_t ad = smem_desc(asm_, kTileM * 16, 128);
          uint64_t bd = smem_desc(w_s + (uint32_t)(width * k0 * 2 + l * width * width * 2), width * 16, 128);
          for (int k = 0; k < width / 16; k += 3, ad += 768, bd += 3 * bstep)
            umma_f16_x3_w(dcol, ad, bd, idesc, k != 0, 256, bstep);
          umma_commit_w(mdone);
        }
      } else if (!last) {
        fence_async_smem();
        tc_fence_before();
        named_bar_sync(1 + g, 128);
        if (issuer) {
          TRC(20 + l, t);
          tc_fence_after();
          uint64_t ad = smem_desc(asm_, kTileM * 16, 128);
          if (a.wstream) {
            w_mma_run(dcol, ad, idesc, 0u, width / 16);
            TRC(30 + l, t);
          } else {
            uint64_t bd = smem_desc(w_s + (uint32_t)(width * k0 * 2 + l * width * width * 2), width * 16, 128);
            int k = 0;
            for (; k + 3 <= width / 16; k += 3, ad += 768, bd += 3 * bstep)
              umma_f16_x3(dcol, ad, bd, idesc, k != 0, 256, bstep);
            for (; k < width / 16; ++k, ad += 256, bd += bstep) umma_f16(dcol, ad, bd, idesc, k != 0);
            TRC(30 + l, t);
          }
          umma_commit(mdone);
        }
      }
    }
    if (issuer) TRC(9, t);
    // ------------------------------------------------ outputs
    if (p >= tile.count) return;
    const int64_t pos = tile.first + p;
    const int64_t id = a.idx ? a.idx[pos] : pos;
#pragma unroll
    for (int k = 0; k < kMaxOut; ++k)
      if (k < out_dim) y[k] = y[k] + s_headb[k];
    if (a.out_mode == OUT_RAW) {
#pragma unroll
      for (int k = 0; k < kMaxOut; ++k)
        if (k < out_dim) a.out_raw[id * out_dim + k] = y[k];
      return;
    }
    double gwt = 1.0;
    if (a.src_kind != SRC_NORM_F32) {
      const int64_t sid = a.gather ? a.gather[id] : id;
      double c3[3];
      point_centre(a.src_kind, a.src, sid, c3);
      gwt = gate_weight(s_exp.cell, a.subdomain_size, a.halo, c3, inv2h);
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
      return;
    }
    const bool covered = den > 0.0;
    if (covered && den != 1.0) {  // a single covering expert has den == 1 (x / 1 == x): skip the f64 divides
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
  };

  // ---- rounds: engine g takes tile base + g; tiles of one round that need
  // different nets run as consecutive sub-rounds around a weight switch
  for (int base = t_begin; base < t_end; base += E) {
    const int lim = min(E, t_end - base);
    int k = 0;
    while (k < lim) {
      const Tile tk = tile_at(base + k);
      if (tk.count <= 0) {
        ++k;
        continue;
      }
      int k2 = k + 1;
      while (k2 < lim) {
        const Tile u = tile_at(base + k2);
        if (u.count > 0 && u.net != tk.net) break;
        ++k2;
      }
      if (tk.net != loaded) load_net(tk.net);
      const Tile mine = (g >= k && g < k2) ? tile_at(base + g) : Tile{};
      if (g >= k && g < k2 && mine.count > 0) {
        if (wait_start && base == t_begin) mbar_wait(bars + 1 + 8 * g + kSlots + 1, 0);
        process(mine, base + g);
      } else if (a.wstream && issuer) {
        w_skip_tile();
      }
      k = k2;
    }
  }

  // ------------------------------------------------ teardown
  if (a.wstream) {  // prefetched weight chunks nobody will use: let the copies land
    __syncthreads();
    if (tid == 0)
      for (uint32_t pos = wcons; pos < s_wnext; ++pos) mbar_wait(wfull + pos % (uint32_t)WR, (pos / WR) & 1u);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem_base, 512);
}
#endif  // NVDB_MLP_KERNEL_TU

}  // namespace nvdb
