// Upper-tree coordinate -> node lookup (K1): VdbGrid.get_values with kind
// (grid.py:310-390) as a bitmask/popcount traversal of the flattened tree.
//
// The reference sorts rows by root key and level-2 slot and resolves groups;
// each row's result is a pure function of its coordinate, so here every
// thread resolves its rows independently:
//   root key (binary search) -> level-2 child bit (tile?) -> popcount rank ->
//   level-1 child bit (tile?) -> popcount rank -> leaf value + active bit.
// Integer-only; the traffic is the coordinate read plus a few L2-resident
// node words per query.
#include <algorithm>
#include <vector>

#include "tree.cuh"

using namespace nvdb;

namespace {

__device__ __forceinline__ int cmp3(const int32_t* k, int x, int y, int z) {
  if (k[0] != x) return k[0] < x ? -1 : 1;
  if (k[1] != y) return k[1] < y ? -1 : 1;
  if (k[2] != z) return k[2] < z ? -1 : 1;
  return 0;
}

__global__ void k_lookup(TreeView t, const int32_t* __restrict__ coords, int64_t n, float* __restrict__ value,
                         uint8_t* __restrict__ active, uint8_t* __restrict__ kind, int32_t* __restrict__ leaf_out) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    const int x = __ldg(coords + 3 * i), y = __ldg(coords + 3 * i + 1), z = __ldg(coords + 3 * i + 2);
    float v = t.background;
    uint8_t a = 0, k = 0;
    int32_t leaf = -1;
    // root: two's-complement masking (grid.py:74-94)
    const int rx = x & ~4095, ry = y & ~4095, rz = z & ~4095;
    int lo = 0, hi = t.nroots - 1, r = -1;
    while (lo <= hi) {
      const int mid = (lo + hi) >> 1;
      const int c = cmp3(t.root_keys + 3 * mid, rx, ry, rz);
      if (c == 0) { r = mid; break; }
      if (c < 0) lo = mid + 1; else hi = mid - 1;
    }
    if (r >= 0) {
      const int n2 = t.root_l2[r];
      if (n2 < 0) {
        v = t.root_tile_value[r];
        a = t.root_tile_active[r];
        k = 1;
      } else {
        const int i2 = (((x & 4095) >> 7) << 10) | (((y & 4095) >> 7) << 5) | ((z & 4095) >> 7);
        const int64_t s2 = (int64_t)n2 * 32768 + i2;
        const int n1 = __ldg(t.l2_slot + s2);
        if (n1 < 0) {
          v = __ldg(t.l2_tiles + s2);
          a = (__ldg(reinterpret_cast<const unsigned long long*>(t.l2_active) + (s2 >> 6)) >> (i2 & 63)) & 1ull;
          k = 1;
        } else {
          const int i1 = (((x & 127) >> 3) << 8) | (((y & 127) >> 3) << 4) | ((z & 127) >> 3);
          const int64_t s1 = (int64_t)n1 * 4096 + i1;
          leaf = __ldg(t.l1_slot + s1);
          if (leaf < 0) {
            v = __ldg(t.l1_tiles + s1);
            a = (__ldg(reinterpret_cast<const unsigned long long*>(t.l1_active) + (s1 >> 6)) >> (i1 & 63)) & 1ull;
            k = 1;
          } else {
            const int i0 = ((x & 7) << 6) | ((y & 7) << 3) | (z & 7);
            v = __ldg(t.leaf_values + (int64_t)leaf * 512 + i0);
            a = (__ldg(reinterpret_cast<const unsigned long long*>(t.leaf_active) + (int64_t)leaf * 8 + (i0 >> 6)) >>
                 (i0 & 63)) & 1ull;
            k = 2;
          }
        }
      }
    }
    value[i] = v;
    active[i] = a;
    kind[i] = k;
    if (leaf_out) leaf_out[i] = leaf;
  }
}

// slot -> child index (node base + set child bits before the slot), -1 for a tile slot
__global__ void k_slot_table(const uint64_t* __restrict__ words, int64_t nslots, int log2_spn,
                             const uint16_t* __restrict__ prefix, const int32_t* __restrict__ base,
                             int32_t* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nslots) return;
  const int64_t node = i >> log2_spn;
  const uint64_t w = words[i >> 6];
  const uint64_t b = 1ull << (i & 63);
  out[i] = (w & b) ? base[node] + prefix[i >> 6] + __popcll(w & (b - 1)) : -1;
}

// exclusive per-node prefix of set child bits, word granularity
__global__ void k_prefix(const uint64_t* __restrict__ words, int64_t nnodes, int wpn, uint16_t* __restrict__ prefix) {
  const int64_t node = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (node >= nnodes) return;
  uint32_t acc = 0;
  for (int w = 0; w < wpn; ++w) {
    prefix[node * wpn + w] = (uint16_t)acc;
    acc += __popcll(words[node * wpn + w]);
  }
}

template <class T>
int upload(nvdb_tree* t, T** dst, const T* src, size_t count) {
  const size_t bytes = sizeof(T) * std::max<size_t>(count, 1);
  NVDB_CUDA_TRY(cudaMalloc(dst, bytes));
  t->owned[t->nowned++] = *dst;
  if (count && src) NVDB_CUDA_TRY(cudaMemcpy(*dst, src, sizeof(T) * count, cudaMemcpyDefault));
  else NVDB_CUDA_TRY(cudaMemset(*dst, 0, bytes));
  return NVDB_OK;
}

}  // namespace

namespace nvdb {

int tree_build_prefix(nvdb_tree* t, cudaStream_t st) {
  if (t->n2 > 0) {
    k_prefix<<<(t->n2 + 127) / 128, 128, 0, st>>>(t->l2_child, t->n2, 512, t->l2_prefix);
    NVDB_CHECK_LAUNCH();
  }
  if (t->n1 > 0) {
    k_prefix<<<(t->n1 + 127) / 128, 128, 0, st>>>(t->l1_child, t->n1, 64, t->l1_prefix);
    NVDB_CHECK_LAUNCH();
  }
  if (t->n2 > 0) {
    const int64_t ns = (int64_t)t->n2 * 32768;
    k_slot_table<<<(int)((ns + 255) / 256), 256, 0, st>>>(t->l2_child, ns, 15, t->l2_prefix, t->l2_child_base,
                                                           t->l2_slot);
    NVDB_CHECK_LAUNCH();
  }
  if (t->n1 > 0) {
    const int64_t ns = (int64_t)t->n1 * 4096;
    k_slot_table<<<(int)((ns + 255) / 256), 256, 0, st>>>(t->l1_child, ns, 12, t->l1_prefix, t->l1_child_base,
                                                           t->l1_slot);
    NVDB_CHECK_LAUNCH();
  }
  return NVDB_OK;
}

int launch_lookup(const nvdb_tree* t, const int32_t* coords, int64_t n, float* value, uint8_t* active, uint8_t* kind,
                  int32_t* leaf, cudaStream_t st) {
  if (n <= 0) return NVDB_OK;
  const int threads = 256;
  const int64_t want = (n + threads - 1) / threads;
  const int blocks = (int)std::min<int64_t>(want, (int64_t)num_sms() * 16);
  k_lookup<<<blocks, threads, 0, st>>>(view_of(t), coords, n, value, active, kind, leaf);
  NVDB_CHECK_LAUNCH();
  return NVDB_OK;
}

}  // namespace nvdb

extern "C" int nvdb_tree_create(const nvdb_tree_desc* d, nvdb_tree** out) {
  if (!d || !out) return fail(NVDB_EINVAL, "nvdb_tree_create: null argument");
  if (d->nroots < 0 || d->n2 < 0 || d->n1 < 0 || d->nl < 0) return fail(NVDB_EINVAL, "negative node count");
  // roots must be sorted for the binary search
  for (int r = 1; r < d->nroots; ++r) {
    const int32_t* a = d->root_keys + 3 * (r - 1);
    const int32_t* b = d->root_keys + 3 * r;
    if (!std::lexicographical_compare(a, a + 3, b, b + 3))
      return fail(NVDB_EINVAL, "root keys must be strictly ascending");
  }
  nvdb_tree* t = new nvdb_tree();
  t->background = d->background;
  t->nroots = d->nroots;
  t->n2 = d->n2;
  t->n1 = d->n1;
  t->nl = d->nl;
  int rc = NVDB_OK;
  auto chk = [&](int r) {
    if (r && !rc) rc = r;
  };
  chk(upload(t, &t->root_keys, d->root_keys, (size_t)3 * d->nroots));
  chk(upload(t, &t->root_l2, d->root_l2, (size_t)d->nroots));
  chk(upload(t, &t->root_tile_value, d->root_tile_value, (size_t)d->nroots));
  chk(upload(t, &t->root_tile_active, d->root_tile_active, (size_t)d->nroots));
  chk(upload(t, &t->l2_child, d->l2_child, (size_t)512 * d->n2));
  chk(upload(t, &t->l2_active, d->l2_active, (size_t)512 * d->n2));
  chk(upload(t, &t->l2_tiles, d->l2_tiles, (size_t)32768 * d->n2));
  chk(upload(t, &t->l2_child_base, d->l2_child_base, (size_t)d->n2));
  chk(upload(t, &t->l2_prefix, (const uint16_t*)nullptr, (size_t)512 * d->n2));
  chk(upload(t, &t->l1_child, d->l1_child, (size_t)64 * d->n1));
  chk(upload(t, &t->l1_active, d->l1_active, (size_t)64 * d->n1));
  chk(upload(t, &t->l1_tiles, d->l1_tiles, (size_t)4096 * d->n1));
  chk(upload(t, &t->l1_child_base, d->l1_child_base, (size_t)d->n1));
  chk(upload(t, &t->l1_prefix, (const uint16_t*)nullptr, (size_t)64 * d->n1));
  chk(upload(t, &t->l2_slot, (const int32_t*)nullptr, (size_t)32768 * d->n2));
  chk(upload(t, &t->l1_slot, (const int32_t*)nullptr, (size_t)4096 * d->n1));
  chk(upload(t, &t->leaf_active, d->leaf_active, (size_t)8 * d->nl));
  chk(upload(t, &t->leaf_values, d->leaf_values, (size_t)512 * d->nl));
  if (d->leaf_patched) chk(upload(t, &t->leaf_patched, d->leaf_patched, (size_t)8 * d->nl));
  if (!rc) rc = tree_build_prefix(t, 0);
  if (!rc && cudaDeviceSynchronize() != cudaSuccess) rc = fail(NVDB_ECUDA, "tree prefix build failed");
  if (rc) {
    nvdb_tree_destroy(t);
    return rc;
  }
  *out = t;
  return NVDB_OK;
}

extern "C" int nvdb_tree_destroy(nvdb_tree* t) {
  if (!t) return NVDB_OK;
  for (int i = 0; i < t->nowned; ++i) cudaFree(t->owned[i]);
  delete t;
  return NVDB_OK;
}

extern "C" int nvdb_lookup(const nvdb_tree* t, const int32_t* coords, int64_t n, float* value, uint8_t* active,
                           uint8_t* kind, int32_t* leaf, void* stream) {
  if (!t) return fail(NVDB_EINVAL, "nvdb_lookup: null tree");
  if (n < 0 || (n > 0 && (!coords || !value || !active || !kind)))
    return fail(NVDB_EINVAL, "nvdb_lookup: bad buffers");
  return launch_lookup(t, coords, n, value, active, kind, leaf, static_cast<cudaStream_t>(stream));
}
