// NVGR byte emission of a decoded grid on the device:
// the level-1 node records and leaf records of gridfile.serialize_grid
// (gridfile.py:43-76) written straight from the dense-leaf decode output, so
// the grid reaches the host as its serialized bytes in one copy instead of
// through ~10^6 Python node objects.
//
// Record layouts (little endian, packed, gridfile.py:5-13):
//   level-1 node: origin i32 x 3 | child mask 512 B | active mask 512 B | 4096 f32 tiles
//   leaf:         origin i32 x 3 | active mask 64 B | 512 f32 values
// Masks are packbits(bits, bitorder="little"): bit i of the stream = slot i.
// Record offsets are arbitrary (the stream is byte packed), so each thread
// produces one ALIGNED 4-byte output word, assembling its bytes from the
// record image, and stores it whole (bytes at a record's two ends are stored
// singly so neighbouring records are not touched).
#include <algorithm>

#include "common.cuh"

using namespace nvdb;

namespace {

constexpr int64_t kLeafRec = 12 + 64 + 2048;
constexpr int64_t kL1Rec = 12 + 512 + 512 + 16384;

struct LeafSrc {
  const int32_t* origins;  // (nl, 3)
  const uint64_t* words;   // (nl, 8) active mask words
  const float* values;     // (nl, 512)
};

struct L1Src {
  const int32_t* origins;  // (n1, 3), decode node order
  const uint8_t* cls;      // (n1, 4096) 0 child / 1 active tile / 2 inactive tile
  const float* tiles;      // (n1, 4096)
};

__device__ __forceinline__ uint32_t leaf_byte(const LeafSrc& s, int64_t r, int k) {
  if (k < 12) return (uint32_t)(s.origins[3 * r + (k >> 2)] >> (8 * (k & 3))) & 0xFFu;
  if (k < 76) {
    const int b = k - 12;
    return (uint32_t)(s.words[8 * r + (b >> 3)] >> (8 * (b & 7))) & 0xFFu;
  }
  const int b = k - 76;
  return (__float_as_uint(s.values[512 * r + (b >> 2)]) >> (8 * (b & 3))) & 0xFFu;
}

__device__ __forceinline__ uint32_t l1_byte(const L1Src& s, int64_t r, int k) {
  if (k < 12) return (uint32_t)(s.origins[3 * r + (k >> 2)] >> (8 * (k & 3))) & 0xFFu;
  if (k < 12 + 1024) {
    const int b = k - 12;
    const uint8_t want = b < 512 ? 0 : 1;  // child mask, then active mask
    const uint8_t* c = s.cls + 4096 * r + 8 * (b & 511);
    uint32_t v = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) v |= (uint32_t)(c[j] == want) << j;
    return v;
  }
  const int b = k - (12 + 1024);
  return (__float_as_uint(s.tiles[4096 * r + (b >> 2)]) >> (8 * (b & 3))) & 0xFFu;
}

// one block row of threads per record chunk: record r covers output bytes
// [off[r], off[r] + len); thread -> aligned word w of that range
template <typename Src, int64_t LEN, uint32_t (*BYTE)(const Src&, int64_t, int)>
__global__ void k_emit(Src src, const int64_t* __restrict__ rec_off, int64_t nrec, uint8_t* __restrict__ out) {
  const int64_t words_per_rec = LEN / 4 + 2;
  const int64_t total = nrec * words_per_rec;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = t / words_per_rec;
    const int64_t w = t - r * words_per_rec;
    const int64_t off = rec_off[r];
    const int64_t a0 = (off & ~3LL) + 4 * w;  // aligned output word
    if (a0 >= off + LEN) continue;
    if (a0 >= off && a0 + 4 <= off + LEN) {
      const int k = (int)(a0 - off);
      const uint32_t v = BYTE(src, r, k) | (BYTE(src, r, k + 1) << 8) | (BYTE(src, r, k + 2) << 16) |
                         (BYTE(src, r, k + 3) << 24);
      *reinterpret_cast<uint32_t*>(out + a0) = v;
    } else {
      for (int j = 0; j < 4; ++j) {
        const int64_t a = a0 + j;
        if (a >= off && a < off + LEN) out[a] = (uint8_t)BYTE(src, r, (int)(a - off));
      }
    }
  }
}

inline int grid_for(int64_t work) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((work + 255) / 256, (int64_t)num_sms() * 16));
}

}  // namespace

extern "C" int nvdb_nvgr_leaf_records(const int32_t* leaf_origins, const uint64_t* active_words, const float* values,
                                      int64_t nl, const int64_t* rec_off, uint8_t* out, void* stream) {
  if (nl < 0 || (nl > 0 && (!leaf_origins || !active_words || !values || !rec_off || !out)))
    return fail(NVDB_EINVAL, "nvdb_nvgr_leaf_records: bad args");
  if (!nl) return NVDB_OK;
  LeafSrc s{leaf_origins, active_words, values};
  k_emit<LeafSrc, kLeafRec, leaf_byte><<<grid_for(nl * (kLeafRec / 4 + 2)), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      s, rec_off, nl, out);
  NVDB_CHECK_LAUNCH();
  return NVDB_OK;
}

extern "C" int nvdb_nvgr_l1_records(const int32_t* node_origins, const uint8_t* l1_class, const float* tiles,
                                    int64_t n1, const int64_t* rec_off, uint8_t* out, void* stream) {
  if (n1 < 0 || (n1 > 0 && (!node_origins || !l1_class || !tiles || !rec_off || !out)))
    return fail(NVDB_EINVAL, "nvdb_nvgr_l1_records: bad args");
  if (!n1) return NVDB_OK;
  L1Src s{node_origins, l1_class, tiles};
  k_emit<L1Src, kL1Rec, l1_byte><<<grid_for(n1 * (kL1Rec / 4 + 2)), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      s, rec_off, n1, out);
  NVDB_CHECK_LAUNCH();
  return NVDB_OK;
}
