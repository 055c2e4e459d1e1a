// Device-resident flattened [Hash,5,4,3] upper tree + leaves (grid.py:248-390).
#pragma once
#include <cstdint>

#include "common.cuh"

struct nvdb_tree {
  float background = 0.f;
  int32_t nroots = 0, n2 = 0, n1 = 0, nl = 0;
  // all device pointers; `owned` buffers are freed by nvdb_tree_destroy
  int32_t* root_keys = nullptr;      // (nroots,3) sorted lexicographically
  int32_t* root_l2 = nullptr;        // (nroots)
  float* root_tile_value = nullptr;  // (nroots)
  uint8_t* root_tile_active = nullptr;
  uint64_t* l2_child = nullptr;      // (n2,512)
  uint64_t* l2_active = nullptr;
  float* l2_tiles = nullptr;         // (n2,32768)
  int32_t* l2_child_base = nullptr;  // (n2)
  uint16_t* l2_prefix = nullptr;     // (n2,512) set child bits before each word
  uint64_t* l1_child = nullptr;      // (n1,64)
  uint64_t* l1_active = nullptr;
  float* l1_tiles = nullptr;         // (n1,4096)
  int32_t* l1_child_base = nullptr;  // (n1)
  uint16_t* l1_prefix = nullptr;     // (n1,64)
  int32_t* l2_slot = nullptr;        // (n2,32768) level-1 node index of a child slot, -1 for a tile
  int32_t* l1_slot = nullptr;        // (n1,4096) leaf index of a child slot, -1 for a tile
  uint64_t* leaf_active = nullptr;   // (nl,8)
  float* leaf_values = nullptr;      // (nl,512)
  uint64_t* leaf_patched = nullptr;  // (nl,8) optional: voxels whose value is an exact patch
  // lookup entries, one 8-byte word per slot / voxel so a lookup makes ONE
  // random L2 sector access per level: [31:0] child index or value bits,
  // [32] active, [34:33] kind (0 child, 1 tile, 2 leaf voxel)
  uint64_t* l2_ent = nullptr;        // (n2,32768)
  uint64_t* l1_ent = nullptr;        // (n1,4096)
  uint64_t* leaf_ent = nullptr;      // (nl,512)
  uint64_t* root_ent = nullptr;      // (nroots) level-2 node index, or the root tile as a kind-1 entry
  void* owned[32] = {};
  int nowned = 0;
};

namespace nvdb {

struct TreeView {  // kernel-side copy of the pointers
  float background;
  int32_t nroots;
  const int32_t* root_keys;
  const int32_t* root_l2;
  const float* root_tile_value;
  const uint8_t* root_tile_active;
  const uint64_t* l2_child;
  const uint64_t* l2_active;
  const float* l2_tiles;
  const int32_t* l2_child_base;
  const uint16_t* l2_prefix;
  const uint64_t* l1_child;
  const uint64_t* l1_active;
  const float* l1_tiles;
  const int32_t* l1_child_base;
  const uint16_t* l1_prefix;
  const int32_t* l2_slot;
  const int32_t* l1_slot;
  const uint64_t* leaf_active;
  const float* leaf_values;
  const uint64_t* l2_ent;
  const uint64_t* l1_ent;
  const uint64_t* leaf_ent;
  const uint64_t* root_ent;
};

inline TreeView view_of(const nvdb_tree* t) {
  return TreeView{t->background,    t->nroots,        t->root_keys,     t->root_l2,   t->root_tile_value,
                  t->root_tile_active, t->l2_child,   t->l2_active,     t->l2_tiles,  t->l2_child_base,
                  t->l2_prefix,     t->l1_child,      t->l1_active,     t->l1_tiles,  t->l1_child_base,
                  t->l1_prefix,     t->l2_slot,       t->l1_slot,       t->leaf_active, t->leaf_values,
                  t->l2_ent,        t->l1_ent,        t->leaf_ent,  t->root_ent};
}

constexpr uint64_t kEntActive = 1ull << 32;
constexpr int kEntKindShift = 33;
constexpr uint64_t kEntMiss = 3ull << kEntKindShift;  // outside every root: background, kind 0

__device__ __forceinline__ int cmp3(const int32_t* k, int x, int y, int z) {
  if (k[0] != x) return k[0] < x ? -1 : 1;
  if (k[1] != y) return k[1] < y ? -1 : 1;
  if (k[2] != z) return k[2] < z ? -1 : 1;
  return 0;
}

// VdbGrid.get_value with kind (grid.py:288-307, 310-390) of one coordinate:
// root key (binary search over the sorted roots, two's-complement masking
// as grid.py:74-94) -> level-2 entry -> level-1 entry -> leaf-voxel entry,
// one dependent 8-byte load per level.  kind 0 outside every node
// (background), 1 tile, 2 leaf voxel; leaf = leaf index or -1.
__device__ __forceinline__ void tree_resolve(const TreeView& t, int x, int y, int z, float& v, uint8_t& a,
                                             uint8_t& k, int32_t& leaf) {
  v = t.background;
  a = 0;
  k = 0;
  leaf = -1;
  const int rx = x & ~4095, ry = y & ~4095, rz = z & ~4095;
  int lo = 0, hi = t.nroots - 1, r = -1;
  while (lo <= hi) {
    const int mid = (lo + hi) >> 1;
    const int c = cmp3(t.root_keys + 3 * mid, rx, ry, rz);
    if (c == 0) {
      r = mid;
      break;
    }
    if (c < 0) lo = mid + 1;
    else hi = mid - 1;
  }
  if (r < 0) return;
  const int n2 = __ldg(t.root_l2 + r);
  if (n2 < 0) {
    v = __ldg(t.root_tile_value + r);
    a = __ldg(t.root_tile_active + r);
    k = 1;
    return;
  }
  const int i2 = (((x & 4095) >> 7) << 10) | (((y & 4095) >> 7) << 5) | ((z & 4095) >> 7);
  uint64_t e = __ldg(reinterpret_cast<const unsigned long long*>(t.l2_ent) + (int64_t)n2 * 32768 + i2);
  if (e >> kEntKindShift) {
    v = __uint_as_float((uint32_t)e);
    a = (uint8_t)((e >> 32) & 1u);
    k = 1;
    return;
  }
  const int i1 = (((x & 127) >> 3) << 8) | (((y & 127) >> 3) << 4) | ((z & 127) >> 3);
  e = __ldg(reinterpret_cast<const unsigned long long*>(t.l1_ent) + (int64_t)(uint32_t)e * 4096 + i1);
  if (e >> kEntKindShift) {
    v = __uint_as_float((uint32_t)e);
    a = (uint8_t)((e >> 32) & 1u);
    k = 1;
    return;
  }
  leaf = (int32_t)(uint32_t)e;
  const int i0 = ((x & 7) << 6) | ((y & 7) << 3) | (z & 7);
  e = __ldg(reinterpret_cast<const unsigned long long*>(t.leaf_ent) + (int64_t)leaf * 512 + i0);
  v = __uint_as_float((uint32_t)e);
  a = (uint8_t)((e >> 32) & 1u);
  k = 2;
}

// computes l2_prefix / l1_prefix and the slot -> child index tables on the
// device (after masks are in place)
int tree_build_prefix(nvdb_tree* t, cudaStream_t st);
int launch_lookup(const nvdb_tree* t, const int32_t* coords, int64_t n, float* value, uint8_t* active,
                  uint8_t* kind, int32_t* leaf, cudaStream_t st);

}  // namespace nvdb
