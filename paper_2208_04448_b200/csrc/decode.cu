// Whole-volume decode helpers (K6): the device side of decoder._reconstruct /
// _fill_leaves (decoder.py:101-211) and HybridGrid.query (decoder.py:239-264).
//
// The host (Python) sequences these primitives exactly like the reference:
//   classify all level-1 slots (nvdb_eval, OUT_L1CLASS)
//   -> level-1 patches, inactive tile values        (nvdb_l1_apply)
//   -> active tiles: select + tile regressor + scatter
//   -> leaves under child slots                     (nvdb_select_u8 + nvdb_leaf_list)
//   -> classify all leaf voxels (nvdb_eval, OUT_L0ACTIVE), level-0 patches
//   -> select active voxels, voxel regressor (OUT_VALUE: clip, scale, background)
//   -> values, patch values, negative fill, packed masks (nvdb_leaf_finalize)
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>
#include <thrust/iterator/transform_iterator.h>

#include <algorithm>

#include "netset.cuh"
#include "tree.cuh"

using namespace nvdb;

namespace {

inline int blocks_for(int64_t n, int threads = 256) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((n + threads - 1) / threads, (int64_t)num_sms() * 32));
}

__global__ void k_l1_apply(uint8_t* cls, float* tiles, const int64_t* patch_slot, const uint8_t* patch_cls,
                           int64_t npatch, const int64_t* tile_slot, const float* tile_value, int64_t ntile,
                           int phase) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (phase == 0) {
    for (int64_t i = i0; i < npatch; i += stride)
      if (patch_slot[i] >= 0) cls[patch_slot[i]] = patch_cls[i];  // < 0: outside every node (flagged)
  } else {
    for (int64_t i = i0; i < ntile; i += stride) {
      const int64_t s = tile_slot[i];
      if (s >= 0 && cls[s] == 2) tiles[s] = tile_value[i];
    }
  }
}

__global__ void k_scatter_f32(float* dst, const int64_t* ids, const float* vals, int64_t n, const int64_t* n_dev,
                              const uint8_t* skip = nullptr) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  if (n_dev) n = min(n, *n_dev);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    const int64_t id = ids[i];
    if (!skip || !skip[id]) dst[id] = vals[i];
  }
}

__global__ void k_fill_i32(int32_t* dst, int64_t n, int32_t v) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) dst[i] = v;
}

__global__ void k_leaf_list(const int64_t* child_slots, int64_t nl, const int32_t* node_origins, int32_t* leaf_origins,
                            int32_t* leaf_of_slot) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nl; i += stride) {
    const int64_t s = child_slots[i];
    const int64_t node = s >> 12;
    const int slot = (int)(s & 4095);
    leaf_origins[3 * i + 0] = node_origins[3 * node + 0] + 8 * (slot >> 8);
    leaf_origins[3 * i + 1] = node_origins[3 * node + 1] + 8 * ((slot >> 4) & 15);
    leaf_origins[3 * i + 2] = node_origins[3 * node + 2] + 8 * (slot & 15);
    if (leaf_of_slot) leaf_of_slot[s] = (int32_t)i;
  }
}

__global__ void k_l0_apply(uint8_t* active, const int64_t* patch_slot, const int32_t* patch_vox,
                           const uint8_t* patch_active, int64_t npatch, const int32_t* leaf_of_slot, int32_t* err) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < npatch; i += stride) {
    const int32_t leaf = patch_slot[i] >= 0 ? leaf_of_slot[patch_slot[i]] : -1;
    if (leaf == -2) continue;  // a leaf owned by another decode shard
    if (leaf < 0) {
      atomicExch(err, 1);  // decoder.py:172-175: patch outside every reconstructed leaf
      continue;
    }
    active[(int64_t)leaf * 512 + patch_vox[i]] = patch_active[i];
  }
}

// values/background, regressed active voxels (phase 0); patches and negative
// fill (phase 1); packed masks (phase 2).  decoder.py:182-210.
__global__ void k_leaf_values(int64_t nl, float background, float* values) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nl * 512; i += stride) values[i] = background;
}

__global__ void k_leaf_patches(const uint8_t* active, const int64_t* patch_slot, const int32_t* patch_vox,
                               const uint8_t* patch_active, const float* patch_value, int64_t npatch,
                               const int32_t* leaf_of_slot, float* values, uint8_t* patched) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < npatch; i += stride) {
    if (!patch_active[i] || patch_slot[i] < 0) continue;
    const int32_t leaf = leaf_of_slot[patch_slot[i]];
    if (leaf < 0) continue;
    const int64_t v = (int64_t)leaf * 512 + patch_vox[i];
    values[v] = patch_value[i];
    if (patched) patched[v] = 1;
  }
}

__global__ void k_leaf_negfill(const uint8_t* active, const int64_t* neg_slot, const uint64_t* neg_bits, int64_t nneg,
                               const int32_t* leaf_of_slot, float neg_value, float* values) {
  // one thread per (entry, voxel)
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nneg * 512; t += stride) {
    const int64_t e = t >> 9;
    const int v = (int)(t & 511);
    if (neg_slot[e] < 0) continue;
    const int32_t leaf = leaf_of_slot[neg_slot[e]];
    if (leaf < 0) continue;
    if (!((neg_bits[e * 8 + (v >> 6)] >> (v & 63)) & 1ull)) continue;
    const int64_t idx = (int64_t)leaf * 512 + v;
    if (!active[idx]) values[idx] = neg_value;
  }
}

__global__ void k_pack_eq(const uint8_t* v, int64_t nwords, uint8_t value, uint64_t* words) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < nwords; w += stride) {
    const uint4* p = reinterpret_cast<const uint4*>(v + w * 64);
    uint64_t bits = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint4 x = p[q];
      const uint32_t xs[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int b = 0; b < 4; ++b)
          if (((xs[j] >> (8 * b)) & 0xFF) == value) bits |= 1ull << (q * 16 + j * 4 + b);
    }
    words[w] = bits;
  }
}

__global__ void k_query_finalize(const int64_t* rows, int64_t nrows, const float* regressed, const int32_t* coords,
                                 const int32_t* leaf, const uint64_t* leaf_patched, const float* leaf_values,
                                 float* value, const int64_t* nrows_dev) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  if (nrows_dev) nrows = min(nrows, *nrows_dev);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nrows; i += stride) {
    const int64_t r = rows[i];
    float v = regressed[i];
    if (leaf_patched) {
      const int32_t lf = leaf[r];
      const int x = coords[3 * r], y = coords[3 * r + 1], z = coords[3 * r + 2];
      const int i0 = ((x & 7) << 6) | ((y & 7) << 3) | (z & 7);
      if ((leaf_patched[(int64_t)lf * 8 + (i0 >> 6)] >> (i0 & 63)) & 1ull) v = leaf_values[(int64_t)lf * 512 + i0];
    }
    value[r] = v;
  }
}

// rows with active && kind == 2 (decoder.py:243)
__global__ void k_neural_rows(const uint8_t* active, const uint8_t* kind, int64_t n, uint8_t* flag) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride)
    flag[i] = (active[i] && kind[i] == 2) ? 1 : 0;
}

struct EqValue {
  uint8_t v;
  __host__ __device__ bool operator()(const uint8_t& x) const { return x == v; }
};

}  // namespace

static int eval_impl(const nvdb_netset* ns, int32_t tag, int32_t src_kind, const void* src, const int64_t* gather,
                     int64_t n, const int64_t* n_dev, const nvdb_eval_out* out, void* ws, size_t ws_bytes,
                     void* stream) {
  if (!ns || !out || tag < 0 || tag > 3 || src_kind < 0 || src_kind > 4) return fail(NVDB_EINVAL, "nvdb_eval: bad args");
  if (n < 0 || (n > 0 && !src)) return fail(NVDB_EINVAL, "nvdb_eval: bad source");
  BlendOut o{};
  o.out_mode = out->out_mode;
  o.out_raw = out->raw;
  o.out_probs = out->probs;
  o.out_u8 = out->u8;
  o.out_f32 = out->f32;
  o.value_scale = out->value_scale;
  o.background = out->background;
  o.clip = out->clip;
  switch (o.out_mode) {
    case OUT_RAW: if (!o.out_raw && n) return fail(NVDB_EINVAL, "nvdb_eval: raw output missing"); break;
    case OUT_PROBS: if ((!o.out_probs || !o.out_u8) && n) return fail(NVDB_EINVAL, "nvdb_eval: probs output missing"); break;
    case OUT_L1CLASS:
    case OUT_L0ACTIVE: if (!o.out_u8 && n) return fail(NVDB_EINVAL, "nvdb_eval: u8 output missing"); break;
    case OUT_VALUE: if (!o.out_f32 && n) return fail(NVDB_EINVAL, "nvdb_eval: f32 output missing"); break;
    default: return fail(NVDB_EINVAL, "nvdb_eval: bad out_mode %d", o.out_mode);
  }
  return run_blended(ns, tag, src_kind, src, gather, n, o, ws, ws_bytes, static_cast<cudaStream_t>(stream), n_dev);
}

extern "C" int nvdb_eval(const nvdb_netset* ns, int32_t tag, int32_t src_kind, const void* src, const int64_t* gather,
                         int64_t n, const nvdb_eval_out* out, void* ws, size_t ws_bytes, void* stream) {
  return eval_impl(ns, tag, src_kind, src, gather, n, nullptr, out, ws, ws_bytes, stream);
}

extern "C" int nvdb_eval_counted(const nvdb_netset* ns, int32_t tag, int32_t src_kind, const void* src,
                                 const int64_t* gather, int64_t capacity, const int64_t* count_dev,
                                 const nvdb_eval_out* out, void* ws, size_t ws_bytes, void* stream) {
  if (!count_dev) return fail(NVDB_EINVAL, "nvdb_eval_counted: count_dev missing");
  return eval_impl(ns, tag, src_kind, src, gather, capacity, count_dev, out, ws, ws_bytes, stream);
}

extern "C" size_t nvdb_select_workspace_bytes(int64_t n) {
  size_t bytes = 0;
  cub::DeviceSelect::Flagged(nullptr, bytes, thrust::counting_iterator<int64_t>(0),
                             thrust::make_transform_iterator((const uint8_t*)nullptr, EqValue{0}), (int64_t*)nullptr,
                             (int64_t*)nullptr, std::max<int64_t>(n, 1));
  return bytes + 256;
}

extern "C" int nvdb_select_u8(const uint8_t* v, int64_t n, uint8_t value, int64_t* ids, int64_t* count, void* ws,
                              size_t ws_bytes, void* stream) {
  if (n < 0 || !count || (n > 0 && (!v || !ids))) return fail(NVDB_EINVAL, "nvdb_select_u8: bad args");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (n == 0) {
    NVDB_CUDA_TRY(cudaMemsetAsync(count, 0, sizeof(int64_t), st));
    return NVDB_OK;
  }
  size_t need = 0;
  thrust::counting_iterator<int64_t> it(0);
  auto flags = thrust::make_transform_iterator(v, EqValue{value});
  cub::DeviceSelect::Flagged(nullptr, need, it, flags, ids, count, n, st);
  if (ws_bytes < need || !ws) return fail(NVDB_ENOMEM, "nvdb_select_u8: workspace %zu < %zu", ws_bytes, need);
  NVDB_CUDA_TRY(cub::DeviceSelect::Flagged(ws, need, it, flags, ids, count, n, st));
  return NVDB_OK;
}

extern "C" int nvdb_l1_apply(uint8_t* cls, float* tiles, int64_t nslots, const int64_t* patch_slot,
                             const uint8_t* patch_cls, int64_t npatch, const int64_t* tile_slot, const float* tile_value,
                             int64_t ntile, void* stream) {
  if (!cls || !tiles || nslots < 0 || npatch < 0 || ntile < 0) return fail(NVDB_EINVAL, "nvdb_l1_apply: bad args");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (npatch) {
    k_l1_apply<<<blocks_for(npatch), 256, 0, st>>>(cls, tiles, patch_slot, patch_cls, npatch, tile_slot, tile_value,
                                                   ntile, 0);
    NVDB_CHECK_LAUNCH();
  }
  if (ntile) {
    k_l1_apply<<<blocks_for(ntile), 256, 0, st>>>(cls, tiles, patch_slot, patch_cls, npatch, tile_slot, tile_value,
                                                  ntile, 1);
    NVDB_CHECK_LAUNCH();
  }
  return NVDB_OK;
}

extern "C" int nvdb_scatter_f32(float* dst, const int64_t* ids, const float* vals, int64_t n, void* stream) {
  if (n < 0 || (n > 0 && (!dst || !ids || !vals))) return fail(NVDB_EINVAL, "nvdb_scatter_f32: bad args");
  if (!n) return NVDB_OK;
  k_scatter_f32<<<blocks_for(n), 256, 0, static_cast<cudaStream_t>(stream)>>>(dst, ids, vals, n, nullptr);
  NVDB_CHECK_LAUNCH();
  return NVDB_OK;
}

// node index of a coordinate through a dense table over the bounding box of
// the level-1 origins (>> 7), then node * 4096 + idx1 and idx0 (grid.py:74-94)
__global__ void k_node_slots(const int32_t* __restrict__ lut, int lx, int ly, int lz, int sx, int sy, int sz,
                             const int32_t* __restrict__ coords, int64_t n, int64_t* __restrict__ slot,
                             int32_t* __restrict__ vox, int32_t* __restrict__ err) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    const int x = coords[3 * i], y = coords[3 * i + 1], z = coords[3 * i + 2];
    const int cx = (x >> 7) - lx, cy = (y >> 7) - ly, cz = (z >> 7) - lz;
    int node = -1;
    if ((unsigned)cx < (unsigned)sx && (unsigned)cy < (unsigned)sy && (unsigned)cz < (unsigned)sz)
      node = lut[((int64_t)cx * sy + cy) * sz + cz];
    const int i1 = (((x & 127) >> 3) << 8) | (((y & 127) >> 3) << 4) | ((z & 127) >> 3);
    slot[i] = node < 0 ? -1 : (int64_t)node * 4096 + i1;
    if (vox) vox[i] = ((x & 7) << 6) | ((y & 7) << 3) | (z & 7);
    if (node < 0 && err) atomicExch(err, 1);
  }
}

extern "C" int nvdb_node_slots(const int32_t* lut, const int32_t* lut_lo, const int32_t* lut_span,
                               const int32_t* coords, int64_t n, int64_t* slot, int32_t* vox, int32_t* err,
                               void* stream) {
  if (n < 0 || !lut_lo || !lut_span || (n > 0 && (!lut || !coords || !slot)))
    return fail(NVDB_EINVAL, "nvdb_node_slots: bad args");
  if (!n) return NVDB_OK;
  k_node_slots<<<blocks_for(n), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      lut, lut_lo[0], lut_lo[1], lut_lo[2], lut_span[0], lut_span[1], lut_span[2], coords, n, slot, vox, err);
  NVDB_CHECK_LAUNCH();
  return NVDB_OK;
}

extern "C" int nvdb_leaf_list(const int64_t* child_slots, int64_t nl, const int32_t* node_origins, int64_t nslots,
                              int32_t* leaf_origins, int32_t* leaf_of_slot, void* stream) {
  if (nl < 0 || nslots < 0 || (nl > 0 && (!child_slots || !node_origins || !leaf_origins)))
    return fail(NVDB_EINVAL, "nvdb_leaf_list: bad args");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (leaf_of_slot && nslots) {
    k_fill_i32<<<blocks_for(nslots), 256, 0, st>>>(leaf_of_slot, nslots, -1);
    NVDB_CHECK_LAUNCH();
  }
  if (nl) {
    k_leaf_list<<<blocks_for(nl), 256, 0, st>>>(child_slots, nl, node_origins, leaf_origins, leaf_of_slot);
    NVDB_CHECK_LAUNCH();
  }
  return NVDB_OK;
}

extern "C" int nvdb_l0_apply(uint8_t* active, const int64_t* patch_slot, const int32_t* patch_vox,
                             const uint8_t* patch_active, int64_t npatch, const int32_t* leaf_of_slot, int32_t* err,
                             void* stream) {
  if (npatch < 0 || (npatch > 0 && (!active || !patch_slot || !patch_vox || !patch_active || !leaf_of_slot || !err)))
    return fail(NVDB_EINVAL, "nvdb_l0_apply: bad args");
  if (!npatch) return NVDB_OK;
  k_l0_apply<<<blocks_for(npatch), 256, 0, static_cast<cudaStream_t>(stream)>>>(active, patch_slot, patch_vox,
                                                                               patch_active, npatch, leaf_of_slot, err);
  NVDB_CHECK_LAUNCH();
  return NVDB_OK;
}

static int leaf_finalize(int64_t nl, const uint8_t* active, const int64_t* act_ids, const float* act_vals,
                         int64_t nact, const int64_t* nact_dev, const int64_t* patch_slot, const int32_t* patch_vox,
                         const uint8_t* patch_active, const float* patch_value, int64_t npatch,
                         const int64_t* neg_slot, const uint64_t* neg_bits, int64_t nneg,
                         const int32_t* leaf_of_slot, float background, float neg_value, float* values,
                         uint64_t* active_words, uint8_t* patched, void* stream) {
  if (nl < 0 || nact < 0 || npatch < 0 || nneg < 0) return fail(NVDB_EINVAL, "nvdb_leaf_finalize: bad counts");
  if (nl == 0) return NVDB_OK;
  if (!active || !values) return fail(NVDB_EINVAL, "nvdb_leaf_finalize: null buffers");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  k_leaf_values<<<blocks_for(nl * 512), 256, 0, st>>>(nl, background, values);
  NVDB_CHECK_LAUNCH();
  if (patched) NVDB_CUDA_TRY(cudaMemsetAsync(patched, 0, (size_t)nl * 512, st));
  if (nact && act_vals) {
    k_scatter_f32<<<blocks_for(nact), 256, 0, st>>>(values, act_ids, act_vals, nact, nact_dev);
    NVDB_CHECK_LAUNCH();
  }
  if (npatch) {
    k_leaf_patches<<<blocks_for(npatch), 256, 0, st>>>(active, patch_slot, patch_vox, patch_active, patch_value,
                                                       npatch, leaf_of_slot, values, patched);
    NVDB_CHECK_LAUNCH();
  }
  if (nneg) {
    k_leaf_negfill<<<blocks_for(nneg * 512), 256, 0, st>>>(active, neg_slot, neg_bits, nneg, leaf_of_slot, neg_value,
                                                           values);
    NVDB_CHECK_LAUNCH();
  }
  if (active_words) {
    k_pack_eq<<<blocks_for(nl * 8), 256, 0, st>>>(active, nl * 8, 1, active_words);
    NVDB_CHECK_LAUNCH();
  }
  return NVDB_OK;
}

extern "C" int nvdb_leaf_finalize(int64_t nl, const uint8_t* active, const int64_t* act_ids, const float* act_vals,
                                  int64_t nact, const int64_t* patch_slot, const int32_t* patch_vox,
                                  const uint8_t* patch_active, const float* patch_value, int64_t npatch,
                                  const int64_t* neg_slot, const uint64_t* neg_bits, int64_t nneg,
                                  const int32_t* leaf_of_slot, float background, float neg_value, float* values,
                                  uint64_t* active_words, uint8_t* patched, void* stream) {
  return leaf_finalize(nl, active, act_ids, act_vals, nact, nullptr, patch_slot, patch_vox, patch_active, patch_value,
                       npatch, neg_slot, neg_bits, nneg, leaf_of_slot, background, neg_value, values, active_words,
                       patched, stream);
}

extern "C" int nvdb_leaf_finalize_counted(int64_t nl, const uint8_t* active, const int64_t* act_ids,
                                          const float* act_vals, int64_t act_capacity, const int64_t* nact_dev,
                                          const int64_t* patch_slot, const int32_t* patch_vox,
                                          const uint8_t* patch_active, const float* patch_value, int64_t npatch,
                                          const int64_t* neg_slot, const uint64_t* neg_bits, int64_t nneg,
                                          const int32_t* leaf_of_slot, float background, float neg_value,
                                          float* values, uint64_t* active_words, uint8_t* patched, void* stream) {
  if (!nact_dev) return fail(NVDB_EINVAL, "nvdb_leaf_finalize_counted: nact_dev missing");
  return leaf_finalize(nl, active, act_ids, act_vals, act_capacity, nact_dev, patch_slot, patch_vox, patch_active,
                       patch_value, npatch, neg_slot, neg_bits, nneg, leaf_of_slot, background, neg_value, values,
                       active_words, patched, stream);
}

extern "C" int nvdb_scatter_f32_counted(float* dst, const int64_t* ids, const float* vals, int64_t capacity,
                                        const int64_t* count_dev, void* stream) {
  if (capacity < 0 || !count_dev || (capacity > 0 && (!dst || !ids || !vals)))
    return fail(NVDB_EINVAL, "nvdb_scatter_f32_counted: bad args");
  if (!capacity) return NVDB_OK;
  k_scatter_f32<<<blocks_for(capacity), 256, 0, static_cast<cudaStream_t>(stream)>>>(dst, ids, vals, capacity,
                                                                                     count_dev);
  NVDB_CHECK_LAUNCH();
  return NVDB_OK;
}

extern "C" int nvdb_scatter_f32_unpatched_counted(float* dst, const int64_t* ids, const float* vals, int64_t capacity,
                                                  const int64_t* count_dev, const uint8_t* skip, void* stream) {
  if (capacity < 0 || !count_dev || (capacity > 0 && (!dst || !ids || !vals || !skip)))
    return fail(NVDB_EINVAL, "nvdb_scatter_f32_unpatched_counted: bad args");
  if (!capacity) return NVDB_OK;
  k_scatter_f32<<<blocks_for(capacity), 256, 0, static_cast<cudaStream_t>(stream)>>>(dst, ids, vals, capacity,
                                                                                     count_dev, skip);
  NVDB_CHECK_LAUNCH();
  return NVDB_OK;
}

extern "C" int nvdb_pack_eq(const uint8_t* v, int64_t nwords, uint8_t value, uint64_t* words, void* stream) {
  if (nwords < 0 || (nwords > 0 && (!v || !words))) return fail(NVDB_EINVAL, "nvdb_pack_eq: bad args");
  if (!nwords) return NVDB_OK;
  k_pack_eq<<<blocks_for(nwords), 256, 0, static_cast<cudaStream_t>(stream)>>>(v, nwords, value, words);
  NVDB_CHECK_LAUNCH();
  return NVDB_OK;
}

extern "C" int nvdb_neural_rows(const uint8_t* active, const uint8_t* kind, int64_t n, uint8_t* flag, void* stream) {
  if (n < 0 || (n > 0 && (!active || !kind || !flag))) return fail(NVDB_EINVAL, "nvdb_neural_rows: bad args");
  if (!n) return NVDB_OK;
  k_neural_rows<<<blocks_for(n), 256, 0, static_cast<cudaStream_t>(stream)>>>(active, kind, n, flag);
  NVDB_CHECK_LAUNCH();
  return NVDB_OK;
}

extern "C" int nvdb_query_finalize(const int64_t* rows, int64_t nrows, const float* regressed, const int32_t* coords,
                                   const int32_t* leaf, const nvdb_tree* tree, float* value, void* stream) {
  if (nrows < 0 || !tree || (nrows > 0 && (!rows || !regressed || !coords || !leaf || !value)))
    return fail(NVDB_EINVAL, "nvdb_query_finalize: bad args");
  if (!nrows) return NVDB_OK;
  k_query_finalize<<<blocks_for(nrows), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      rows, nrows, regressed, coords, leaf, tree->leaf_patched, tree->leaf_values, value, nullptr);
  NVDB_CHECK_LAUNCH();
  return NVDB_OK;
}

extern "C" int nvdb_query_finalize_counted(const int64_t* rows, int64_t capacity, const int64_t* nrows_dev,
                                           const float* regressed, const int32_t* coords, const int32_t* leaf,
                                           const nvdb_tree* tree, float* value, void* stream) {
  if (capacity < 0 || !tree || !nrows_dev || (capacity > 0 && (!rows || !regressed || !coords || !leaf || !value)))
    return fail(NVDB_EINVAL, "nvdb_query_finalize_counted: bad args");
  if (!capacity) return NVDB_OK;
  k_query_finalize<<<blocks_for(capacity), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      rows, capacity, regressed, coords, leaf, tree->leaf_patched, tree->leaf_values, value, nrows_dev);
  NVDB_CHECK_LAUNCH();
  return NVDB_OK;
}
