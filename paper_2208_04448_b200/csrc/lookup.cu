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
#include <cstring>
#include <vector>

#include "tree.cuh"

using namespace nvdb;

namespace {

constexpr int kRootLinear = 16;  // roots staged in shared memory (and scanned linearly) up to this count

// Level-synchronous resolve of Q queries (tree_resolve's result for each):
// every level's Q entry loads are issued back to back (predicated, no
// early exits), so a thread keeps Q independent random loads in flight per
// level instead of one dependent chain.  Root keys / entries come from
// shared memory when the block staged them (s_keys != nullptr); larger
// root tables take the binary search in global memory.
template <int Q>
__device__ __forceinline__ void resolve_q(const TreeView& t, const int32_t* s_keys, const uint64_t* s_rent,
                                          const int (&x)[Q], const int (&y)[Q], const int (&z)[Q], float (&v)[Q],
                                          uint8_t (&a)[Q], uint8_t (&k)[Q], int32_t (&lf)[Q]) {
  uint64_t e[Q];
  if (s_keys && t.nroots <= kRootLinear) {
    // few roots (the common case): branch-free scan of the staged keys
#pragma unroll
    for (int j = 0; j < Q; ++j) {
      const int rx = x[j] & ~4095, ry = y[j] & ~4095, rz = z[j] & ~4095;
      e[j] = kEntMiss;
      for (int r = 0; r < t.nroots; ++r)
        if (s_keys[3 * r] == rx && s_keys[3 * r + 1] == ry && s_keys[3 * r + 2] == rz) e[j] = s_rent[r];
    }
  } else {
#pragma unroll
    for (int j = 0; j < Q; ++j) {
      const int rx = x[j] & ~4095, ry = y[j] & ~4095, rz = z[j] & ~4095;
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
      e[j] = r < 0 ? kEntMiss : __ldg(reinterpret_cast<const unsigned long long*>(t.root_ent) + r);
    }
  }
#pragma unroll
  for (int j = 0; j < Q; ++j) {  // level 2
    const int i2 = (((x[j] & 4095) >> 7) << 10) | (((y[j] & 4095) >> 7) << 5) | ((z[j] & 4095) >> 7);
    if ((e[j] >> kEntKindShift) == 0)
      e[j] = __ldg(reinterpret_cast<const unsigned long long*>(t.l2_ent) + (int64_t)(uint32_t)e[j] * 32768 + i2);
  }
#pragma unroll
  for (int j = 0; j < Q; ++j) {  // level 1
    const int i1 = (((x[j] & 127) >> 3) << 8) | (((y[j] & 127) >> 3) << 4) | ((z[j] & 127) >> 3);
    if ((e[j] >> kEntKindShift) == 0)
      e[j] = __ldg(reinterpret_cast<const unsigned long long*>(t.l1_ent) + (int64_t)(uint32_t)e[j] * 4096 + i1);
  }
#pragma unroll
  for (int j = 0; j < Q; ++j) {  // leaf voxel
    const int i0 = ((x[j] & 7) << 6) | ((y[j] & 7) << 3) | (z[j] & 7);
    lf[j] = -1;
    if ((e[j] >> kEntKindShift) == 0) {
      lf[j] = (int32_t)(uint32_t)e[j];
      e[j] = __ldg(reinterpret_cast<const unsigned long long*>(t.leaf_ent) + (int64_t)lf[j] * 512 + i0);
    }
  }
#pragma unroll
  for (int j = 0; j < Q; ++j) {
    const uint32_t kd = (uint32_t)(e[j] >> kEntKindShift);
    const bool miss = kd == 3u;
    v[j] = miss ? t.background : __uint_as_float((uint32_t)e[j]);
    a[j] = miss ? 0 : (uint8_t)((e[j] >> 32) & 1u);
    k[j] = miss ? 0 : (uint8_t)kd;
  }
}


// Neural rows of a query batch (decoder.py:243: active && kind == 2) appended
// by the lookup itself: rows whose voxel carries an exact patch keep the
// value just looked up (what the reference's finalize writes) and are only
// counted; the others go to rows[] for the regressor.  One atomic per warp
// per iteration (warp-aggregated); the row order is not deterministic, the
// values are (each row is evaluated and written independently).
struct RowSink {
  int64_t* rows;                 // (n) capacity
  unsigned long long* count;     // rows appended
  unsigned long long* npatched;  // neural rows answered by an exact patch
  const uint64_t* patched;       // tree leaf_patched (nullable)
};

template <int Q>
__device__ __forceinline__ void append_rows(const RowSink& s, const int64_t (&id)[Q], const bool (&nr)[Q],
                                            const int32_t (&lf)[Q], const int (&x)[Q], const int (&y)[Q],
                                            const int (&z)[Q]) {
  bool app[Q];
  int npt = 0;
#pragma unroll
  for (int j = 0; j < Q; ++j) {
    bool pt = false;
    if (nr[j] && s.patched) {
      const int i0 = ((x[j] & 7) << 6) | ((y[j] & 7) << 3) | (z[j] & 7);
      pt = (__ldg(reinterpret_cast<const unsigned long long*>(s.patched) + (int64_t)lf[j] * 8 + (i0 >> 6)) >>
            (i0 & 63)) & 1ull;
    }
    app[j] = nr[j] && !pt;
    npt += (nr[j] && pt) ? 1 : 0;
  }
  const unsigned m = __activemask();
  const int lane = threadIdx.x & 31, leader = __ffs(m) - 1;
  const unsigned lt = (1u << lane) - 1u;
  unsigned bal[Q];
  int tot = 0;
#pragma unroll
  for (int j = 0; j < Q; ++j) {
    bal[j] = __ballot_sync(m, app[j]);
    tot += __popc(bal[j]);
  }
  for (int o = 16; o > 0; o >>= 1) npt += __shfl_xor_sync(m, npt, o);  // inactive lanes contribute 0
  unsigned long long base = 0;
  if (lane == leader) {
    if (tot) base = atomicAdd(s.count, (unsigned long long)tot);
    if (npt) atomicAdd(s.npatched, (unsigned long long)npt);
  }
  base = __shfl_sync(m, base, leader);
  int off = 0;
#pragma unroll
  for (int j = 0; j < Q; ++j) {
    if (app[j]) s.rows[base + off + __popc(bal[j] & lt)] = id[j];
    off += __popc(bal[j]);
  }
}

// Four queries per thread: three 16-byte coordinate loads (the thread's 48
// contiguous bytes), one level-synchronous resolve, then one 16-byte value
// store, one 4-byte active store and one 4-byte kind store.  ROWS: the
// neural rows are appended to a RowSink instead of writing leaf indices.
template <bool ROWS>
__global__ void __launch_bounds__(256) k_lookup(TreeView t, const int32_t* __restrict__ coords, int64_t n,
                                                float* __restrict__ value, uint8_t* __restrict__ active,
                                                uint8_t* __restrict__ kind, int32_t* __restrict__ leaf_out,
                                                RowSink sink) {
  __shared__ int32_t s_keys[3 * kRootLinear];
  __shared__ uint64_t s_rent[kRootLinear];
  const bool staged = t.nroots <= kRootLinear;
  if (staged) {
    for (int i = threadIdx.x; i < 3 * t.nroots; i += blockDim.x) s_keys[i] = t.root_keys[i];
    for (int i = threadIdx.x; i < t.nroots; i += blockDim.x) s_rent[i] = t.root_ent[i];
    __syncthreads();
  }
  const int32_t* sk = staged ? s_keys : nullptr;
  const uint64_t* sr = staged ? s_rent : nullptr;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t nq4 = n >> 2;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nq4; q += stride) {
    const int4* cp = reinterpret_cast<const int4*>(coords + 12 * q);
    const int4 c0 = __ldcs(cp), c1 = __ldcs(cp + 1), c2 = __ldcs(cp + 2);
    const int xs[4] = {c0.x, c0.w, c1.z, c2.y}, ys[4] = {c0.y, c1.x, c1.w, c2.z}, zs[4] = {c0.z, c1.y, c2.x, c2.w};
    float v[4];
    uint8_t a[4], k[4];
    int32_t lf[4];
    resolve_q<4>(t, sk, sr, xs, ys, zs, v, a, k, lf);
    __stcs(reinterpret_cast<float4*>(value) + q, make_float4(v[0], v[1], v[2], v[3]));
    __stcs(reinterpret_cast<unsigned int*>(active) + q,
           (uint32_t)a[0] | ((uint32_t)a[1] << 8) | ((uint32_t)a[2] << 16) | ((uint32_t)a[3] << 24));
    __stcs(reinterpret_cast<unsigned int*>(kind) + q,
           (uint32_t)k[0] | ((uint32_t)k[1] << 8) | ((uint32_t)k[2] << 16) | ((uint32_t)k[3] << 24));
    if constexpr (ROWS) {
      const int64_t id[4] = {4 * q, 4 * q + 1, 4 * q + 2, 4 * q + 3};
      const bool nr[4] = {a[0] && k[0] == 2, a[1] && k[1] == 2, a[2] && k[2] == 2, a[3] && k[3] == 2};
      append_rows<4>(sink, id, nr, lf, xs, ys, zs);
    } else if (leaf_out) {
      __stcs(reinterpret_cast<int4*>(leaf_out) + q, make_int4(lf[0], lf[1], lf[2], lf[3]));
    }
  }
  // tail (n % 4 rows)
  const int64_t i = 4 * nq4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) {
    float v;
    uint8_t a, k;
    int32_t lf;
    const int x = coords[3 * i], y = coords[3 * i + 1], z = coords[3 * i + 2];
    tree_resolve(t, x, y, z, v, a, k, lf);
    value[i] = v;
    active[i] = a;
    kind[i] = k;
    if constexpr (ROWS) {
      const int64_t id[1] = {i};
      const bool nr[1] = {a && k == 2};
      const int32_t lfa[1] = {lf};
      const int xa[1] = {x}, ya[1] = {y}, za[1] = {z};
      append_rows<1>(sink, id, nr, lfa, xa, ya, za);
    } else if (leaf_out) {
      leaf_out[i] = lf;
    }
  }
}

// scalar form for buffers that are not 16-byte aligned
__global__ void k_lookup1(TreeView t, const int32_t* __restrict__ coords, int64_t n, float* __restrict__ value,
                          uint8_t* __restrict__ active, uint8_t* __restrict__ kind, int32_t* __restrict__ leaf_out) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    float v;
    uint8_t a, k;
    int32_t lf;
    tree_resolve(t, __ldg(coords + 3 * i), __ldg(coords + 3 * i + 1), __ldg(coords + 3 * i + 2), v, a, k, lf);
    value[i] = v;
    active[i] = a;
    kind[i] = k;
    if (leaf_out) leaf_out[i] = lf;
  }
}

// packed lookup entries of one level: child index, or tile value + active bit
__global__ void k_pack_level(const int32_t* __restrict__ slot, const float* __restrict__ tiles,
                             const uint64_t* __restrict__ active, int64_t nslots, uint64_t* __restrict__ ent) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nslots) return;
  const int32_t c = slot[i];
  if (c >= 0) {
    ent[i] = (uint64_t)(uint32_t)c;
  } else {
    const uint64_t act = (active[i >> 6] >> (i & 63)) & 1ull;
    ent[i] = (uint64_t)__float_as_uint(tiles[i]) | (act << 32) | (1ull << kEntKindShift);
  }
}

__global__ void k_pack_leaf(const float* __restrict__ values, const uint64_t* __restrict__ active, int64_t nvox,
                            uint64_t* __restrict__ ent) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nvox) return;
  const uint64_t act = (active[i >> 6] >> (i & 63)) & 1ull;
  ent[i] = (uint64_t)__float_as_uint(values[i]) | (act << 32) | (2ull << kEntKindShift);
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
  if (t->n2 > 0) {
    const int64_t ns = (int64_t)t->n2 * 32768;
    k_pack_level<<<(int)((ns + 255) / 256), 256, 0, st>>>(t->l2_slot, t->l2_tiles, t->l2_active, ns, t->l2_ent);
    NVDB_CHECK_LAUNCH();
  }
  if (t->n1 > 0) {
    const int64_t ns = (int64_t)t->n1 * 4096;
    k_pack_level<<<(int)((ns + 255) / 256), 256, 0, st>>>(t->l1_slot, t->l1_tiles, t->l1_active, ns, t->l1_ent);
    NVDB_CHECK_LAUNCH();
  }
  if (t->nl > 0) {
    const int64_t nv = (int64_t)t->nl * 512;
    k_pack_leaf<<<(int)((nv + 255) / 256), 256, 0, st>>>(t->leaf_values, t->leaf_active, nv, t->leaf_ent);
    NVDB_CHECK_LAUNCH();
  }
  return NVDB_OK;
}

int launch_lookup(const nvdb_tree* t, const int32_t* coords, int64_t n, float* value, uint8_t* active, uint8_t* kind,
                  int32_t* leaf, cudaStream_t st) {
  if (n <= 0) return NVDB_OK;
  const int threads = 256;
  const bool aligned = ((reinterpret_cast<uintptr_t>(coords) | reinterpret_cast<uintptr_t>(value) |
                         reinterpret_cast<uintptr_t>(leaf)) & 15) == 0 &&
                       ((reinterpret_cast<uintptr_t>(active) | reinterpret_cast<uintptr_t>(kind)) & 3) == 0;
  if (aligned) {
    const int64_t want = (std::max<int64_t>(n / 4, 1) + threads - 1) / threads;
    const int blocks = (int)std::min<int64_t>(want, (int64_t)num_sms() * 16);
    k_lookup<false><<<blocks, threads, 0, st>>>(view_of(t), coords, n, value, active, kind, leaf, RowSink{});
  } else {
    const int64_t want = (n + threads - 1) / threads;
    const int blocks = (int)std::min<int64_t>(want, (int64_t)num_sms() * 16);
    k_lookup1<<<blocks, threads, 0, st>>>(view_of(t), coords, n, value, active, kind, leaf);
  }
  NVDB_CHECK_LAUNCH();
  return NVDB_OK;
}

int launch_lookup_rows(const nvdb_tree* t, const int32_t* coords, int64_t n, float* value, uint8_t* active,
                       uint8_t* kind, int64_t* rows, int64_t* count, int64_t* npatched, cudaStream_t st) {
  NVDB_CUDA_TRY(cudaMemsetAsync(count, 0, 8, st));
  NVDB_CUDA_TRY(cudaMemsetAsync(npatched, 0, 8, st));
  if (n <= 0) return NVDB_OK;
  const int threads = 256;
  const int64_t want = (std::max<int64_t>(n / 4, 1) + threads - 1) / threads;
  const int blocks = (int)std::min<int64_t>(want, (int64_t)num_sms() * 16);
  const RowSink sink{rows, reinterpret_cast<unsigned long long*>(count), reinterpret_cast<unsigned long long*>(npatched),
                     t->leaf_patched};
  k_lookup<true><<<blocks, threads, 0, st>>>(view_of(t), coords, n, value, active, kind, nullptr, sink);
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
  chk(upload(t, &t->l2_ent, (const uint64_t*)nullptr, (size_t)32768 * d->n2));
  chk(upload(t, &t->l1_ent, (const uint64_t*)nullptr, (size_t)4096 * d->n1));
  chk(upload(t, &t->leaf_ent, (const uint64_t*)nullptr, (size_t)512 * d->nl));
  {  // root entries: level-2 node index, or the root tile (kind 1, value bits, active bit)
    std::vector<uint64_t> re((size_t)d->nroots);
    for (int r = 0; r < d->nroots; ++r) {
      if (d->root_l2[r] >= 0) {
        re[r] = (uint64_t)(uint32_t)d->root_l2[r];
      } else {
        uint32_t vb;
        std::memcpy(&vb, d->root_tile_value + r, 4);
        re[r] = (uint64_t)vb | ((uint64_t)(d->root_tile_active[r] ? 1 : 0) << 32) | (1ull << kEntKindShift);
      }
    }
    chk(upload(t, &t->root_ent, re.data(), re.size()));
  }
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

extern "C" int nvdb_lookup_rows(const nvdb_tree* t, const int32_t* coords, int64_t n, float* value, uint8_t* active,
                                uint8_t* kind, int64_t* rows, int64_t* count, int64_t* npatched, void* stream) {
  if (!t) return fail(NVDB_EINVAL, "nvdb_lookup_rows: null tree");
  if (n < 0 || !count || !npatched || (n > 0 && (!coords || !value || !active || !kind || !rows)))
    return fail(NVDB_EINVAL, "nvdb_lookup_rows: bad buffers");
  if ((reinterpret_cast<uintptr_t>(coords) | reinterpret_cast<uintptr_t>(value)) & 15 ||
      (reinterpret_cast<uintptr_t>(active) | reinterpret_cast<uintptr_t>(kind)) & 3)
    return fail(NVDB_EINVAL, "nvdb_lookup_rows: coords/value need 16-byte, active/kind 4-byte alignment");
  return launch_lookup_rows(t, coords, n, value, active, kind, rows, count, npatched, static_cast<cudaStream_t>(stream));
}

extern "C" int nvdb_lookup(const nvdb_tree* t, const int32_t* coords, int64_t n, float* value, uint8_t* active,
                           uint8_t* kind, int32_t* leaf, void* stream) {
  if (!t) return fail(NVDB_EINVAL, "nvdb_lookup: null tree");
  if (n < 0 || (n > 0 && (!coords || !value || !active || !kind)))
    return fail(NVDB_EINVAL, "nvdb_lookup: bad buffers");
  return launch_lookup(t, coords, n, value, active, kind, leaf, static_cast<cudaStream_t>(stream));
}
