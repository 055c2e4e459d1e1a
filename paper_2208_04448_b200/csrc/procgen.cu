// Seeded value-noise fBm density on the device: the
// reference's gen_fbm_density (procgen.py:96-171 value noise + fbm, 283-309
// thresholded FOG leaves) evaluated per voxel of every leaf block covering
// the domain, bit-for-bit: f64 lattice hashes and quintic weights, the same
// operation order as numpy (explicit round-to-nearest intrinsics, no FMA
// contraction), f32 storage.  Input plumbing for the C3 workload, not the
// hot path.
#include "common.cuh"

using namespace nvdb;

namespace {

constexpr unsigned long long K1 = 0x9E3779B97F4A7C15ull, K2 = 0xBF58476D1CE4E5B9ull, K3 = 0x94D049BB133111EBull,
                             K4 = 0xD6E8FEB86659FD93ull, K5 = 0xA24BAED4963EE407ull;

__device__ __forceinline__ double lattice(long long ix, long long iy, long long iz, unsigned long long seed) {
  unsigned long long h = ((unsigned long long)ix * K1) ^ ((unsigned long long)iy * K2) ^
                         ((unsigned long long)iz * K3) ^ (seed * K4);
  h ^= h >> 30;
  h *= K2;
  h ^= h >> 27;
  h *= K3;
  h ^= h >> 31;
  return __dmul_rn((double)(h >> 40), 1.0 / (double)(1 << 24));
}

__device__ __forceinline__ double quintic(double t) {  // t * t * t * (t * (t * 6.0 - 15.0) + 10.0)
  const double ttt = __dmul_rn(__dmul_rn(t, t), t);
  const double in = __dadd_rn(__dmul_rn(t, __dsub_rn(__dmul_rn(t, 6.0), 15.0)), 10.0);
  return __dmul_rn(ttt, in);
}

__device__ __forceinline__ double lerp(double a, double b, double w) {  // a + w * (b - a)
  return __dadd_rn(a, __dmul_rn(w, __dsub_rn(b, a)));
}

__device__ double value_noise(double px, double py, double pz, unsigned long long seed) {
  const double fx0 = floor(px), fy0 = floor(py), fz0 = floor(pz);
  const long long ix = (long long)fx0, iy = (long long)fy0, iz = (long long)fz0;
  const double wx = quintic(__dsub_rn(px, (double)ix)), wy = quintic(__dsub_rn(py, (double)iy));
  const double wz = quintic(__dsub_rn(pz, (double)iz));
  const double c000 = lattice(ix, iy, iz, seed), c001 = lattice(ix, iy, iz + 1, seed);
  const double c010 = lattice(ix, iy + 1, iz, seed), c011 = lattice(ix, iy + 1, iz + 1, seed);
  const double c100 = lattice(ix + 1, iy, iz, seed), c101 = lattice(ix + 1, iy, iz + 1, seed);
  const double c110 = lattice(ix + 1, iy + 1, iz, seed), c111 = lattice(ix + 1, iy + 1, iz + 1, seed);
  const double c00 = lerp(c000, c001, wz), c01 = lerp(c010, c011, wz);
  const double c10 = lerp(c100, c101, wz), c11 = lerp(c110, c111, wz);
  const double c0 = lerp(c00, c01, wy), c1 = lerp(c10, c11, wy);
  return lerp(c0, c1, wx);
}

// one thread per voxel of the listed leaf blocks; keep[b] = any active voxel
__global__ void k_fbm_leaves(nvdb_fbm_desc s, const int32_t* __restrict__ origins, int64_t nblocks,
                             float* __restrict__ values, uint8_t* __restrict__ active, int32_t* __restrict__ keep) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nblocks * 512) return;
  const int64_t b = i >> 9;
  const int v = (int)(i & 511);
  const long long x = origins[3 * b] + (v >> 6), y = origins[3 * b + 1] + ((v >> 3) & 7),
                  z = origins[3 * b + 2] + (v & 7);
  const bool inside = x >= s.lo[0] && x <= s.hi[0] && y >= s.lo[1] && y <= s.hi[1] && z >= s.lo[2] && z <= s.hi[2];
  const double px = __dmul_rn((double)x, s.voxel_size), py = __dmul_rn((double)y, s.voxel_size);
  const double pz = __dmul_rn((double)z, s.voxel_size);
  double total = 0.0, amp = 1.0, freq = s.base_frequency, norm = 0.0;
  for (int o = 0; o < s.octaves; ++o) {
    const unsigned long long oseed = s.seed ^ ((unsigned long long)o * K5);
    const double vn = value_noise(__dmul_rn(px, freq), __dmul_rn(py, freq), __dmul_rn(pz, freq), oseed);
    total = __dadd_rn(total, __dmul_rn(amp, vn));
    norm = __dadd_rn(norm, amp);
    amp = __dmul_rn(amp, s.gain);
    freq = __dmul_rn(freq, s.lacunarity);
  }
  double val = __ddiv_rn(total, norm);
  val = fmin(fmax(val, 0.0), 1.0);
  const bool act = inside && val > s.threshold;
  values[i] = act ? __double2float_rn(val) : 0.0f;
  active[i] = act ? 1 : 0;
  if (act) keep[b] = 1;
}

}  // namespace

extern "C" int nvdb_fbm_leaves(const nvdb_fbm_desc* spec, const int32_t* origins, int64_t nblocks, float* values,
                               uint8_t* active, int32_t* keep, void* stream) {
  if (!spec || nblocks < 0 || (nblocks > 0 && (!origins || !values || !active || !keep)))
    return fail(NVDB_EINVAL, "nvdb_fbm_leaves: bad args");
  if (spec->octaves < 1) return fail(NVDB_EINVAL, "octaves must be >= 1");
  if (nblocks == 0) return NVDB_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t n = nblocks * 512;
  k_fbm_leaves<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(*spec, origins, nblocks, values, active, keep);
  NVDB_CHECK_LAUNCH();
  return NVDB_OK;
}
