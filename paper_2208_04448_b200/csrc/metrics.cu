// Verification metrics on the device: the sums behind
// svcodec.metrics.iou / rmse / mcd (metrics.py:116-230) for two grids held
// as device trees, so parity can be checked at C3 / C5 scale where the
// reference's Python metrics do not finish.
//
// One pass enumerates grid A's leaf voxels (and, separately, A's tile
// extents) and resolves each coordinate in grid B with the same lookup as
// nvdb_lookup; the symmetric metrics take two passes (A->B, B->A).  Per pass
// (sums index):
//   0 |act A|             1 |act A & act B|       (FOG IoU; RMSE union)
//   2 |occ A|             3 |occ A & occ B|       (SDF IoU: value <= 0 leaf voxels + tile extents)
//   4 sum_{act A, act B} (vA - vB)^2              (RMSE, counted on the A->B pass only)
//   5 sum_{act A, !act B} (vA - bg_B)^2           (RMSE, both passes)
//   6 surface points of A   7 sum |trilinear_B(p)| over them   (mCD)
// Per-block partials are summed on the host in block order (deterministic).
#include <algorithm>

#include "tree.cuh"

using namespace nvdb;

namespace {

constexpr int kSums = 8;
constexpr int kMetThreads = 256;

struct MetPass {
  TreeView a, b;
  const int32_t* a_leaf_org;  // (nl, 3) A's leaf origins, A's tree order
  int64_t a_nl;
  float bg_b;
  // A's tile extents (host-compacted): origin, extent (8 or 128), value, active
  const int32_t* tile_org;
  const int32_t* tile_ext;
  const float* tile_val;
  const uint8_t* tile_act;
  const int64_t* tile_first;  // prefix of extent^3 (ntiles + 1)
  int64_t ntiles;
};

__device__ __forceinline__ float resolve_value(const TreeView& t, int x, int y, int z, uint8_t* act, uint8_t* kind) {
  float v;
  uint8_t a, k;
  int32_t lf;
  tree_resolve(t, x, y, z, v, a, k, lf);
  if (act) *act = a;
  if (kind) *kind = k;
  return v;
}

// metrics.py:197-215: corner values from ordinary lookups, f64 weights
__device__ double trilinear(const TreeView& t, double px, double py, double pz) {
  const double bx = floor(px), by = floor(py), bz = floor(pz);
  const double fx = px - bx, fy = py - by, fz = pz - bz;
  const int ix = (int)bx, iy = (int)by, iz = (int)bz;
  double out = 0.0;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const int ox = (c >> 2) & 1, oy = (c >> 1) & 1, oz = c & 1;
    const float v = resolve_value(t, ix + ox, iy + oy, iz + oz, nullptr, nullptr);
    double w = 1.0;
    w *= ox ? fx : 1.0 - fx;
    w *= oy ? fy : 1.0 - fy;
    w *= oz ? fz : 1.0 - fz;
    out += w * (double)v;
  }
  return out;
}

__device__ void block_flush(double (&acc)[kSums], double* __restrict__ part) {
  __shared__ double s[kMetThreads / 32][kSums];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < kSums; ++k) {
    double v = acc[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if (lane == 0) s[w][k] = v;
  }
  __syncthreads();
  if (threadIdx.x < kSums) {
    double v = 0.0;
    for (int i = 0; i < kMetThreads / 32; ++i) v += s[i][threadIdx.x];
    part[blockIdx.x * kSums + threadIdx.x] += v;
  }
}

__global__ void __launch_bounds__(kMetThreads) k_metric_leaves(MetPass p, int sdf, int want_mcd, double* part) {
  double acc[kSums] = {0, 0, 0, 0, 0, 0, 0, 0};
  const int64_t nv = p.a_nl * 512;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nv; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t leaf = i >> 9;
    const int v9 = (int)(i & 511);
    const int x = p.a_leaf_org[3 * leaf] + (v9 >> 6), y = p.a_leaf_org[3 * leaf + 1] + ((v9 >> 3) & 7),
              z = p.a_leaf_org[3 * leaf + 2] + (v9 & 7);
    const float va = p.a.leaf_values[i];
    const bool aa = (p.a.leaf_active[i >> 6] >> (i & 63)) & 1ull;
    uint8_t ab, kb;
    const float vb = resolve_value(p.b, x, y, z, &ab, &kb);
    if (aa) {
      acc[0] += 1.0;
      if (ab) {
        acc[1] += 1.0;
        const double d = (double)va - (double)vb;
        acc[4] += d * d;
      } else {
        const double d = (double)va - (double)p.bg_b;
        acc[5] += d * d;
      }
    }
    if (sdf && va <= 0.0f) {
      acc[2] += 1.0;
      if (kb != 0 && vb <= 0.0f) acc[3] += 1.0;
    }
    if (want_mcd && aa) {
      // metrics.py:168-194: +x/+y/+z neighbours in A, zero crossings, exact zeros once
      bool zero_pt = false;
      const double v0 = (double)va;
#pragma unroll
      for (int axis = 0; axis < 3; ++axis) {
        uint8_t na;
        const float nvv = resolve_value(p.a, x + (axis == 0), y + (axis == 1), z + (axis == 2), &na, nullptr);
        if (!na) continue;
        const double v1 = (double)nvv;
        if (v0 * v1 < 0.0) {
          const double t = v0 / (v0 - v1);
          const double px = x + (axis == 0 ? t : 0.0), py = y + (axis == 1 ? t : 0.0),
                       pz = z + (axis == 2 ? t : 0.0);
          acc[6] += 1.0;
          acc[7] += fabs(trilinear(p.b, px, py, pz));
        }
        if (v0 == 0.0) zero_pt = true;
      }
      if (zero_pt) {
        acc[6] += 1.0;
        acc[7] += fabs(trilinear(p.b, (double)x, (double)y, (double)z));
      }
    }
  }
  block_flush(acc, part);
}

// tile extents of A (active tiles for the active sets; non-positive tiles
// for the SDF occupied set), expanded voxel by voxel (metrics.py:45-66, 68-89)
__global__ void __launch_bounds__(kMetThreads) k_metric_tiles(MetPass p, int sdf, double* part) {
  double acc[kSums] = {0, 0, 0, 0, 0, 0, 0, 0};
  const int64_t total = p.ntiles ? p.tile_first[p.ntiles] : 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = p.ntiles - 1;
    while (lo < hi) {  // last tile with first <= i
      const int64_t mid = (lo + hi + 1) >> 1;
      if (p.tile_first[mid] <= i) lo = mid;
      else hi = mid - 1;
    }
    const int64_t r = i - p.tile_first[lo];
    const int e = p.tile_ext[lo];
    const int sh = e == 8 ? 3 : 7;
    const int x = p.tile_org[3 * lo] + (int)(r >> (2 * sh)), y = p.tile_org[3 * lo + 1] + (int)((r >> sh) & (e - 1)),
              z = p.tile_org[3 * lo + 2] + (int)(r & (e - 1));
    const float va = p.tile_val[lo];
    const bool aa = p.tile_act[lo] != 0;
    uint8_t ab, kb;
    const float vb = resolve_value(p.b, x, y, z, &ab, &kb);
    if (aa) {
      acc[0] += 1.0;
      if (ab) {
        acc[1] += 1.0;
        const double d = (double)va - (double)vb;
        acc[4] += d * d;
      } else {
        const double d = (double)va - (double)p.bg_b;
        acc[5] += d * d;
      }
    }
    if (sdf && va <= 0.0f) {
      acc[2] += 1.0;
      if (kb != 0 && vb <= 0.0f) acc[3] += 1.0;
    }
  }
  block_flush(acc, part);
}

}  // namespace

extern "C" size_t nvdb_metric_partials(void) { return (size_t)num_sms() * 4 * kSums; }

extern "C" int nvdb_metric_pass(const nvdb_tree* a, const int32_t* a_leaf_origins, const nvdb_tree* b,
                                const int32_t* tile_origin, const int32_t* tile_extent, const float* tile_value,
                                const uint8_t* tile_active, const int64_t* tile_first, int64_t ntiles, int32_t sdf,
                                int32_t want_mcd, double* partials, void* stream) {
  if (!a || !b || !partials || (a->nl > 0 && !a_leaf_origins) ||
      (ntiles > 0 && (!tile_origin || !tile_extent || !tile_value || !tile_active || !tile_first)))
    return fail(NVDB_EINVAL, "nvdb_metric_pass: bad args");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int blocks = num_sms() * 4;
  NVDB_CUDA_TRY(cudaMemsetAsync(partials, 0, sizeof(double) * (size_t)blocks * kSums, st));
  MetPass p{view_of(a), view_of(b), a_leaf_origins, a->nl, b->background,
            tile_origin, tile_extent, tile_value, tile_active, tile_first, ntiles};
  k_metric_leaves<<<blocks, kMetThreads, 0, st>>>(p, sdf, want_mcd, partials);
  NVDB_CHECK_LAUNCH();
  if (ntiles > 0) {
    k_metric_tiles<<<blocks, kMetThreads, 0, st>>>(p, sdf, partials);
    NVDB_CHECK_LAUNCH();
  }
  return NVDB_OK;
}
