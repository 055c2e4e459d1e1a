// Device-resident set of every expert's networks (the decode/eval "model").
#pragma once
#include <algorithm>
#include <cstdlib>
#include <cstdint>
#include <vector>

#include "common.cuh"
#include "mlp.cuh"

struct nvdb_netset {
  int nnets = 0, nexperts = 0;
  int subdomain_size = 512, halo = 8;
  uint8_t* dev_blob = nullptr;            // weight images + float params
  bool owns_blob = true;                  // false: the caller's buffer (nvdb_netset_create_at)
  nvdb::NetDev* dev_nets = nullptr;       // [nnets]
  nvdb::ExpertDev* dev_experts = nullptr; // [nexperts]
  int32_t* dev_cells = nullptr;           // [nexperts][3] sorted lexicographically (= sid order)
  int32_t* dev_tagnet = nullptr;          // [nexperts][4] net index or -1
  std::vector<nvdb::NetDev> nets;         // host copies (device pointers inside)
  std::vector<nvdb::ExpertDev> experts;
  std::vector<int32_t> tagnet;            // [nexperts][4]
  uint32_t max_wimg = 0;
  int max_width = 16;
  int max_depth = 1;
  int max_k0 = 64;
  int act = 2;  // shared hidden activation of every net
};

namespace nvdb {

// shared-memory plan for an MLP launch over nets with the given maxima
struct SmemPlan {
  uint32_t w_off, region_off, region_bytes, small_off, bar_off, total;
};

inline SmemPlan plan_smem(uint32_t max_wimg, int max_width, int groups = 2) {
  SmemPlan p;
  p.w_off = 0;
  p.region_off = (uint32_t)align_up(max_wimg, 1024);
  const uint32_t feat = 2u * kChunkBytes;
  const uint32_t hid = (uint32_t)kTileM * (uint32_t)max_width * 2u;
  p.region_bytes = (uint32_t)align_up(feat > hid ? feat : hid, 1024);
  p.small_off = p.region_off + (uint32_t)groups * p.region_bytes;  // one region per tile group
  p.bar_off = (uint32_t)align_up(p.small_off + kSmallFloats * 4, 16);
  p.total = p.bar_off + 128;
  return p;
}

constexpr uint32_t kMaxDynSmem = 227 * 1024 - 512;  // leave room for static __shared__

// shared-memory / TMEM plan of mlp_eval_kernel for nets up to the given maxima
struct EvalPlan {
  uint32_t w_off, region_off, region_bytes, small_off, bar_off, total;
  int engines, tcols, ereg, wstream, wring, ok;
  uint32_t wring_off, wslot_bytes;
  int wslack;
  int sm_bias, sm_headw, sm_headb, sm_b2pi, sm_lat, sm_hx;
};

// smem: weights | engines x max(kSlots feature chunks, hidden fp16 A tile) | small params | mbarriers
// TMEM: engines x accumulator of W <= 512 columns
inline EvalPlan plan_eval(uint32_t max_wimg, int W, int depth, int k0, uint32_t limit) {
  EvalPlan p{};
  auto a4 = [](int v) { return (v + 3) & ~3; };
  p.sm_bias = 0;
  p.sm_headw = a4(depth * W);
  p.sm_headb = p.sm_headw + a4(3 * W);
  p.sm_b2pi = p.sm_headb + 4;
  p.sm_lat = p.sm_b2pi + a4(3 * (k0 / 2));
  p.sm_hx = p.sm_lat + a4(4 * k0);  // lattice table: 8 floats per complex feature
  const uint32_t small_bytes = (uint32_t)p.sm_hx * 4u;
  p.w_off = 0;
  p.region_off = (uint32_t)align_up(max_wimg, 1024);
  p.tcols = (W + 15) & ~15;
  const int by_tmem = std::max(0, std::min(kMaxEngines, 512 / std::max(p.tcols, 16)));
  long long base_ereg = (long long)align_up(std::max<size_t>((size_t)kSlots * kEChunkBytes,
                                                                   (size_t)kTileM * W * 2), 1024);
  // resident weights when at least two engines fit beside them, else streamed weights
  long long room = (long long)limit - p.region_off - small_bytes - 16 - 1024;
  p.ereg = (int)base_ereg;
  p.engines = room > 0 ? std::min<int>(by_tmem, (int)std::min<long long>(kMaxEngines, room / base_ereg)) : 0;
  p.wstream = 0;
  p.wring = 0;
  p.wring_off = 0;
  if (p.engines < 2) {
    // streamed: 64 K feature chunks (two 16 KB slots) beside the hidden A tile
    base_ereg = (long long)align_up(std::max<size_t>((size_t)kSlots * kEChunkBytesS, (size_t)kTileM * W * 2), 1024);
    // streamed: as many engines as TMEM allows, then the CTA-wide weight ring:
    // slots of up to 4 K = 16 chunks (W x 32 bytes each), as many slots (2..4)
    // as fit, bigger slots first (the issuer's bookkeeping is per slot)
    p.wstream = 1;
    p.region_off = 0;
    room = (long long)limit - small_bytes - 16 - 1024;
    p.engines = 0;
    for (int ne = by_tmem; ne >= 1 && !p.engines; --ne)
      for (int pc = 4; pc >= 1 && !p.engines; pc /= 2)
        for (int r = 4; r >= 2; --r) {
          if (ne * base_ereg + (long long)r * pc * W * 32 <= room) {
            p.engines = ne;
            p.wring = r;
            p.wslot_bytes = (uint32_t)(pc * W * 32);
            p.ereg = (int)base_ereg;
            break;
          }
        }
    p.wslack = p.wring >= 3 ? 1 : 0;
    p.wring_off = (uint32_t)(p.engines * base_ereg);
  }
  p.region_bytes = (uint32_t)(std::max(p.engines, 1) * p.ereg) +
                   (p.wstream ? (uint32_t)p.wring * p.wslot_bytes : 0u);
  p.small_off = p.region_off + p.region_bytes;
  p.bar_off = (uint32_t)align_up(p.small_off + small_bytes, 16);
  p.total = p.bar_off + 1024;
  p.ok = p.engines >= 1 && p.total <= limit && W % 16 == 0 && W <= 256;
  return p;
}

int launch_mlp(const nvdb_netset* ns, MlpArgs a, const int32_t* npairs_dev, int grid, cudaStream_t st);

// Generic gate-blended evaluation over a point source (all experts owning
// net `tag`), writing `out_mode` outputs.  Workspace from the caller.
struct BlendOut {
  int32_t out_mode;
  float* out_raw;
  double* out_probs;
  uint8_t* out_u8;
  float* out_f32;
  double value_scale;
  float background;
  int32_t clip;
};
size_t blended_workspace_bytes(const nvdb_netset* ns, int64_t n);
int run_blended(const nvdb_netset* ns, int tag, int src_kind, const void* src, const int64_t* gather, int64_t n,
                const BlendOut& o, void* ws, size_t ws_bytes, cudaStream_t st, const int64_t* n_dev = nullptr);

}  // namespace nvdb
