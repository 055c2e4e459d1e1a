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
};

inline TreeView view_of(const nvdb_tree* t) {
  return TreeView{t->background,    t->nroots,        t->root_keys,     t->root_l2,   t->root_tile_value,
                  t->root_tile_active, t->l2_child,   t->l2_active,     t->l2_tiles,  t->l2_child_base,
                  t->l2_prefix,     t->l1_child,      t->l1_active,     t->l1_tiles,  t->l1_child_base,
                  t->l1_prefix,     t->l2_slot,       t->l1_slot,       t->leaf_active, t->leaf_values};
}

// computes l2_prefix / l1_prefix and the slot -> child index tables on the
// device (after masks are in place)
int tree_build_prefix(nvdb_tree* t, cudaStream_t st);
int launch_lookup(const nvdb_tree* t, const int32_t* coords, int64_t n, float* value, uint8_t* active,
                  uint8_t* kind, int32_t* leaf, cudaStream_t st);

}  // namespace nvdb
