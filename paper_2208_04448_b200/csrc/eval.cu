// Netset upload, the forward_block seam and the generic gate-blended
// evaluation driver (inference.py:39-84, partition.py:160-256).
#define NVDB_MLP_KERNEL_TU
#include <immintrin.h>
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "netset.cuh"

using namespace nvdb;

namespace {

uint16_t f2h_bits(float f) {
  __half h = __float2half_rn(f);
  uint16_t b;
  std::memcpy(&b, &h, 2);
  return b;
}

int round_up_i(int v, int a) { return (v + a - 1) / a * a; }

// one weight matrix (rows x cols, row-major fp32, times `scale`) into the fp16
// K-major core-matrix image of R padded rows: 8 consecutive k of a row are 16
// contiguous bytes of the image, converted 8 at a time with F16C when the
// host has it (round to nearest even, as __float2half_rn)
__attribute__((target("avx,f16c"))) void pack_rows_f16c(uint16_t* img, const float* w, int rows, int cols, int R,
                                                        float scale) {
  const __m256 sc = _mm256_set1_ps(scale);
  for (int n = 0; n < rows; ++n) {
    const float* src = w + (size_t)n * cols;
    int k = 0;
    for (; k + 8 <= cols; k += 8) {
      __m256 v = _mm256_loadu_ps(src + k);
      if (scale != 1.0f) v = _mm256_mul_ps(v, sc);
      const __m128i h = _mm256_cvtps_ph(v, _MM_FROUND_TO_NEAREST_INT | _MM_FROUND_NO_EXC);
      _mm_storeu_si128(reinterpret_cast<__m128i*>(img + kmajor_offset(n, k, R) / 2), h);
    }
    for (; k < cols; ++k) img[kmajor_offset(n, k, R) / 2] = f2h_bits(scale == 1.0f ? src[k] : src[k] * scale);
  }
}

void pack_rows(uint16_t* img, const float* w, int rows, int cols, int R, float scale) {
  static const bool f16c = __builtin_cpu_supports("f16c") && __builtin_cpu_supports("avx");
  if (f16c) {
    pack_rows_f16c(img, w, rows, cols, R, scale);
    return;
  }
  for (int n = 0; n < rows; ++n)
    for (int k = 0; k < cols; ++k)
      img[kmajor_offset(n, k, R) / 2] = f2h_bits(scale == 1.0f ? w[(size_t)n * cols + k] : w[(size_t)n * cols + k] * scale);
}

}  // namespace

extern "C" const char* nvdb_last_error(void) { return last_error_slot().c_str(); }
extern "C" int nvdb_version(void) { return 1; }
extern "C" long long nvdb_launch_count(void) { return launch_counter().load(); }

#ifdef NVDB_TRACE
// trace build only (make trace): arm the CTA-0 timeline of mlp_eval_kernel
extern "C" NVDB_API int nvdb_debug_trace(void* buf, uint32_t cap) {
  unsigned long long* p = static_cast<unsigned long long*>(buf);
  const unsigned int zero = 0;
  cudaMemcpyToSymbol(g_trace, &p, sizeof(p));
  cudaMemcpyToSymbol(g_trace_cap, &cap, sizeof(cap));
  cudaMemcpyToSymbol(g_trace_n, &zero, sizeof(zero));
  return cudaDeviceSynchronize() == cudaSuccess ? NVDB_OK : NVDB_ECUDA;
}
#endif

// ---------------------------------------------------------------------------
// netset
// ---------------------------------------------------------------------------
// mem == nullptr: the library allocates (cudaMalloc) and uploads synchronously;
// else the netset lives in the caller's device buffer (`mem_bytes` >= the
// size nvdb_netset_device_bytes reports) and is uploaded on `st` without a
// host synchronisation; *need (nullable) receives the device bytes.
static int netset_create(const nvdb_net_desc* nets, int32_t nnets, const nvdb_expert_desc* experts, int32_t nexperts,
                         int32_t subdomain_size, int32_t halo, void* mem, size_t mem_bytes, cudaStream_t st,
                         nvdb_netset** out, size_t* need) {
  if ((!out && !need) || (nnets > 0 && !nets) || nexperts < 0 || (nexperts > 0 && !experts))
    return fail(NVDB_EINVAL, "nvdb_netset_create: null argument");
  if (subdomain_size <= 0 || subdomain_size % 512 || halo <= 0)
    return fail(NVDB_EINVAL, "bad subdomain size %d / halo %d", subdomain_size, halo);
  if (out) *out = nullptr;
  // ---- host packing: one blob, every piece 256-byte aligned
  struct Piece {
    size_t wimg, bias, headw, headb, b2pi, lat;
  };
  std::vector<Piece> pieces(nnets);
  std::vector<NetDev> hnets(nnets);
  size_t total = 0;
  auto take = [&](size_t bytes) {
    size_t off = total;
    total = align_up(total + bytes, 256);
    return off;
  };
  uint32_t max_wimg = 0;
  int max_width = 16;
  for (int i = 0; i < nnets; ++i) {
    const nvdb_net_desc& d = nets[i];
    if (d.m < 1 || d.depth < 1 || d.width < 1 || (d.out_dim != 1 && d.out_dim != 3))
      return fail(NVDB_EINVAL, "net %d: bad dims m=%d depth=%d width=%d out=%d", i, d.m, d.depth, d.width,
                  d.out_dim);
    if (i > 0 && d.activation != nets[0].activation)
      return fail(NVDB_EUNSUPPORTED, "all nets of a netset must share one hidden activation");
    if (d.head == NVDB_HEAD_LOGITS && d.out_dim != 3)
      return fail(NVDB_EUNSUPPORTED, "net %d: logits head must be 3 wide", i);
    const int W = round_up_i(d.width, 16);
    const int k0 = round_up_i(2 * d.m, kChunkK);
    if (W > 256 || d.depth > 4 || k0 > 1024)
      return fail(NVDB_EUNSUPPORTED, "net %d: width %d depth %d 2m %d exceeds this build (<=256, <=4, <=1024)",
                  i, d.width, d.depth, 2 * d.m);
    NetDev& nd = hnets[i];
    nd.k0 = k0;
    nd.width = W;
    nd.depth = d.depth;
    nd.out_dim = d.out_dim;
    nd.act = d.activation;
    nd.head = d.head;
    nd.expert = 0;
    nd.omega = d.activation == NVDB_ACT_SINE ? d.frequency : 1.0f;
    nd.wimg_bytes = (uint32_t)align_up((size_t)2 * ((size_t)W * k0 + (size_t)(d.depth - 1) * W * W), 16);
    max_wimg = std::max(max_wimg, nd.wimg_bytes);
    max_width = std::max(max_width, W);
    pieces[i].wimg = take(nd.wimg_bytes);
    pieces[i].bias = take(sizeof(float) * d.depth * W);
    pieces[i].headw = take(sizeof(float) * d.out_dim * W);
    pieces[i].headb = take(sizeof(float) * 4);
    pieces[i].b2pi = take(sizeof(float) * 3 * (k0 / 2));
    pieces[i].lat = take(sizeof(float) * k0);
  }
  int max_depth = 1, max_k0 = 64;
  for (int i = 0; i < nnets; ++i) {
    max_depth = std::max(max_depth, hnets[i].depth);
    max_k0 = std::max(max_k0, hnets[i].k0);
  }
  const EvalPlan plan = plan_eval(max_wimg, max_width, max_depth, max_k0, kMaxDynSmem);
  if (!plan.ok)
    return fail(NVDB_EUNSUPPORTED, "nets need %u B of shared memory / %d-wide TMEM accumulators; "
                "weight streaming not built", plan.total, max_width);
  {
    auto al0 = [](size_t x) { return (x + 255) & ~(size_t)255; };
    const size_t need_bytes =
        al0(al0(al0(al0(std::max<size_t>(total, 256)) + sizeof(NetDev) * std::max(nnets, 1)) +
                sizeof(ExpertDev) * std::max(nexperts, 1)) + sizeof(int32_t) * 3 * std::max(nexperts, 1)) +
        sizeof(int32_t) * 4 * std::max(nexperts, 1);
    if (need) *need = need_bytes;
    if (!out) return NVDB_OK;
    if (mem && mem_bytes < need_bytes)
      return fail(NVDB_ENOMEM, "netset needs %zu device bytes, buffer has %zu", need_bytes, mem_bytes);
  }
  std::vector<uint8_t> blob(std::max<size_t>(total, 256), 0);
  for (int i = 0; i < nnets; ++i) {
    const nvdb_net_desc& d = nets[i];
    const NetDev& nd = hnets[i];
    const int W = nd.width, k0 = nd.k0, m = d.m;
    const bool sine = d.activation == NVDB_ACT_SINE;
    const float om = sine ? d.frequency : 1.0f;
    uint16_t* wimg = reinterpret_cast<uint16_t*>(blob.data() + pieces[i].wimg);
    // layer 0: B operand (N = W rows, K = k0), serialized interleaved feature order;
    // the feature amplitude (1 unless set) folded in, omega applied in the
    // fp32 epilogue so 16-bit container weights stay exact in fp16
    pack_rows(wimg, d.weights[0], d.width, 2 * m, W, d.amplitude);
    size_t base = (size_t)W * k0;
    for (int l = 1; l < d.depth; ++l) {
      pack_rows(wimg + base, d.weights[l], d.width, d.width, W, 1.0f);
      base += (size_t)W * W;
    }
    float* bias = reinterpret_cast<float*>(blob.data() + pieces[i].bias);
    for (int l = 0; l < d.depth; ++l)
      for (int n = 0; n < d.width; ++n) bias[l * W + n] = d.biases[l][n] * om;
    float* hw = reinterpret_cast<float*>(blob.data() + pieces[i].headw);
    for (int k = 0; k < d.out_dim; ++k)
      for (int n = 0; n < d.width; ++n) hw[k * W + n] = d.weights[d.depth][(size_t)k * d.width + n];
    float* hb = reinterpret_cast<float*>(blob.data() + pieces[i].headb);
    for (int k = 0; k < d.out_dim; ++k) hb[k] = d.biases[d.depth][k];
    float* b2 = reinterpret_cast<float*>(blob.data() + pieces[i].b2pi);
    for (int ax = 0; ax < 3; ++ax)
      for (int f = 0; f < m; ++f) b2[ax * (k0 / 2) + f] = d.b2pi[ax * m + f];
  }
  // ---- experts: sorted by cell (sid order), tag -> net
  std::vector<ExpertDev> hexp(nexperts);
  std::vector<int32_t> cells(3 * std::max(nexperts, 1)), tagnet(4 * std::max(nexperts, 1), -1);
  for (int e = 0; e < nexperts; ++e) {
    const nvdb_expert_desc& x = experts[e];
    if (e > 0) {
      const int* p = experts[e - 1].cell;
      if (!(std::lexicographical_compare(p, p + 3, x.cell, x.cell + 3)))
        return fail(NVDB_EINVAL, "experts must be in ascending cell (sid) order");
    }
    if (!(x.norm_scale > 0)) return fail(NVDB_EINVAL, "expert %d: norm_scale must be > 0", e);
    for (int i = 0; i < 3; ++i) {
      hexp[e].norm_origin[i] = x.norm_origin[i];
      hexp[e].cell[i] = x.cell[i];
      cells[3 * e + i] = x.cell[i];
    }
    hexp[e].norm_scale = x.norm_scale;
    hexp[e].inv_scale = 1.0 / x.norm_scale;
    for (int t = 0; t < 4; ++t) {
      const int ni = x.net_index[t];
      if (ni >= nnets) return fail(NVDB_EINVAL, "expert %d: net index %d out of range", e, ni);
      tagnet[4 * e + t] = ni;
      if (ni >= 0) hnets[ni].expert = e;
    }
  }
  // lattice step table per net: exp(i * 2 pi b_fy / norm_scale) of its expert
  for (int i = 0; i < nnets; ++i) {
    const nvdb_net_desc& d = nets[i];
    const double nsc = nexperts ? experts[hnets[i].expert].norm_scale : 1.0;
    float* lat = reinterpret_cast<float*>(blob.data() + pieces[i].lat);
    for (int f = 0; f < hnets[i].k0 / 2; ++f) {
      const double beta = f < d.m ? (double)d.b2pi[1 * d.m + f] / nsc : 0.0;
      lat[2 * f] = (float)std::cos(beta);
      lat[2 * f + 1] = (float)std::sin(beta);
    }
  }
  nvdb_netset* ns = new nvdb_netset();
  ns->nnets = nnets;
  ns->nexperts = nexperts;
  ns->subdomain_size = subdomain_size;
  ns->halo = halo;
  ns->max_wimg = max_wimg;
  ns->max_width = max_width;
  ns->max_depth = max_depth;
  ns->max_k0 = max_k0;
  ns->act = nnets ? nets[0].activation : NVDB_ACT_SINE;
  auto cleanup = [&](int code) {
    nvdb_netset_destroy(ns);
    return code;
  };
  // one device allocation and one upload: [blob | nets | experts | cells | tagnet]
  auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
  const size_t off_nets = al(blob.size());
  const size_t off_exp = al(off_nets + sizeof(NetDev) * std::max(nnets, 1));
  const size_t off_cells = al(off_exp + sizeof(ExpertDev) * std::max(nexperts, 1));
  const size_t off_tag = al(off_cells + sizeof(int32_t) * cells.size());
  const size_t all_bytes = off_tag + sizeof(int32_t) * tagnet.size();
  if (mem) {
    ns->dev_blob = static_cast<uint8_t*>(mem);
    ns->owns_blob = false;
  } else if (cudaMalloc(&ns->dev_blob, all_bytes) != cudaSuccess) {
    return cleanup(fail(NVDB_ECUDA, "cudaMalloc netset"));
  }
  ns->dev_nets = reinterpret_cast<NetDev*>(ns->dev_blob + off_nets);
  ns->dev_experts = reinterpret_cast<ExpertDev*>(ns->dev_blob + off_exp);
  ns->dev_cells = reinterpret_cast<int32_t*>(ns->dev_blob + off_cells);
  ns->dev_tagnet = reinterpret_cast<int32_t*>(ns->dev_blob + off_tag);
  for (int i = 0; i < nnets; ++i) {
    hnets[i].wimg = ns->dev_blob + pieces[i].wimg;
    hnets[i].bias = reinterpret_cast<const float*>(ns->dev_blob + pieces[i].bias);
    hnets[i].headw = reinterpret_cast<const float*>(ns->dev_blob + pieces[i].headw);
    hnets[i].headb = reinterpret_cast<const float*>(ns->dev_blob + pieces[i].headb);
    hnets[i].b2pi = reinterpret_cast<const float*>(ns->dev_blob + pieces[i].b2pi);
    hnets[i].lat = reinterpret_cast<const float*>(ns->dev_blob + pieces[i].lat);
  }
  blob.resize(all_bytes, 0);
  if (nnets) std::memcpy(blob.data() + off_nets, hnets.data(), sizeof(NetDev) * nnets);
  if (nexperts) std::memcpy(blob.data() + off_exp, hexp.data(), sizeof(ExpertDev) * nexperts);
  std::memcpy(blob.data() + off_cells, cells.data(), sizeof(int32_t) * cells.size());
  std::memcpy(blob.data() + off_tag, tagnet.data(), sizeof(int32_t) * tagnet.size());
  // pageable source: cudaMemcpyAsync returns once the bytes are staged, so the
  // host vector may go; the upload is ordered on the caller's stream
  if ((mem ? cudaMemcpyAsync(ns->dev_blob, blob.data(), all_bytes, cudaMemcpyHostToDevice, st)
           : cudaMemcpy(ns->dev_blob, blob.data(), all_bytes, cudaMemcpyHostToDevice)) != cudaSuccess)
    return cleanup(fail(NVDB_ECUDA, "upload netset"));
  ns->nets = hnets;
  ns->experts = hexp;
  ns->tagnet = tagnet;
  *out = ns;
  return NVDB_OK;
}

extern "C" int nvdb_netset_create(const nvdb_net_desc* nets, int32_t nnets, const nvdb_expert_desc* experts,
                                  int32_t nexperts, int32_t subdomain_size, int32_t halo, nvdb_netset** out) {
  if (!out) return fail(NVDB_EINVAL, "nvdb_netset_create: null argument");
  return netset_create(nets, nnets, experts, nexperts, subdomain_size, halo, nullptr, 0, nullptr, out, nullptr);
}

extern "C" int nvdb_netset_device_bytes(const nvdb_net_desc* nets, int32_t nnets, const nvdb_expert_desc* experts,
                                        int32_t nexperts, int32_t subdomain_size, int32_t halo, size_t* bytes) {
  if (!bytes) return fail(NVDB_EINVAL, "nvdb_netset_device_bytes: null argument");
  return netset_create(nets, nnets, experts, nexperts, subdomain_size, halo, nullptr, 0, nullptr, nullptr, bytes);
}

extern "C" int nvdb_netset_create_at(const nvdb_net_desc* nets, int32_t nnets, const nvdb_expert_desc* experts,
                                     int32_t nexperts, int32_t subdomain_size, int32_t halo, void* device_mem,
                                     size_t device_bytes, void* stream, nvdb_netset** out) {
  if (!out || !device_mem) return fail(NVDB_EINVAL, "nvdb_netset_create_at: null argument");
  return netset_create(nets, nnets, experts, nexperts, subdomain_size, halo, device_mem, device_bytes,
                       static_cast<cudaStream_t>(stream), out, nullptr);
}

extern "C" int nvdb_netset_destroy(nvdb_netset* ns) {
  if (!ns) return NVDB_OK;
  if (ns->owns_blob) cudaFree(ns->dev_blob);  // the tables live in the same allocation
  delete ns;
  return NVDB_OK;
}

namespace nvdb {

int launch_mlp(const nvdb_netset* ns, MlpArgs a, const int32_t* npairs_dev, int grid, cudaStream_t st) {
  const EvalPlan plan = plan_eval(ns->max_wimg, ns->max_width, ns->max_depth, ns->max_k0, kMaxDynSmem);
  // at least ~120 KB so only one CTA (which owns all 512 TMEM columns) fits per SM
  const uint32_t smem = std::max<uint32_t>(plan.total, 120 * 1024);  // one CTA per SM (owns all TMEM)
  static long long smem_limit = -1;
  if (smem_limit < 0) {
    smem_limit = std::min(std::min(enable_max_smem(mlp_eval_kernel<ACT_RELU>), enable_max_smem(mlp_eval_kernel<ACT_TANH>)),
                          enable_max_smem(mlp_eval_kernel<ACT_SINE>));
    if (smem_limit < 0) return fail(NVDB_ECUDA, "cannot raise shared memory limit of mlp_eval_kernel");
  }
  if ((long long)plan.total > smem_limit)
    return fail(NVDB_EUNSUPPORTED, "MLP kernel needs %u B shared memory, device allows %lld", plan.total, smem_limit);
  a.nets = ns->dev_nets;
  a.experts = ns->dev_experts;
  a.npairs_dev = npairs_dev;
  a.subdomain_size = ns->subdomain_size;
  a.halo = ns->halo;
  a.w_off = plan.w_off;
  a.region_off = plan.region_off;
  a.region_bytes = plan.region_bytes;
  a.small_off = plan.small_off;
  a.bar_off = plan.bar_off;
  a.engines = plan.engines;
  a.tcols = plan.tcols;
  a.ereg = plan.ereg;
  a.wstream = plan.wstream;
  a.wring = plan.wring;
  a.wring_off = plan.wring_off;
  a.wslot_bytes = plan.wslot_bytes;
  a.wslack = plan.wslack;
  a.sm_bias = plan.sm_bias;
  a.sm_headw = plan.sm_headw;
  a.sm_headb = plan.sm_headb;
  a.sm_b2pi = plan.sm_b2pi;
  a.sm_lat = plan.sm_lat;
  a.sm_hx = plan.sm_hx;
  if (grid <= 0) return NVDB_OK;
  switch (ns->act) {
    case ACT_RELU: mlp_eval_kernel<ACT_RELU><<<grid, 128 * plan.engines, smem, st>>>(a); break;
    case ACT_TANH: mlp_eval_kernel<ACT_TANH><<<grid, 128 * plan.engines, smem, st>>>(a); break;
    default: mlp_eval_kernel<ACT_SINE><<<grid, 128 * plan.engines, smem, st>>>(a); break;
  }
  NVDB_CHECK_LAUNCH();
  return NVDB_OK;
}

}  // namespace nvdb

extern "C" int nvdb_forward(const nvdb_netset* ns, int32_t net, const float* pts, int64_t n, float* out,
                            void* stream) {
  if (!ns || net < 0 || net >= ns->nnets) return fail(NVDB_EINVAL, "nvdb_forward: bad netset/net");
  if (n < 0 || (n > 0 && (!pts || !out))) return fail(NVDB_EINVAL, "nvdb_forward: bad buffers");
  if (n == 0) return NVDB_OK;
  MlpArgs a{};
  a.tiles = nullptr;
  a.implicit_net = net;
  a.n_implicit = n;
  const int64_t ntiles = (n + kTileM - 1) / kTileM;
  a.npairs = (int32_t)((ntiles + 1) / 2);
  a.src_kind = SRC_NORM_F32;
  a.src = pts;
  a.out_mode = OUT_RAW;
  a.out_raw = out;
  const int grid = std::min<int64_t>(a.npairs, num_sms());
  return launch_mlp(ns, a, nullptr, grid, static_cast<cudaStream_t>(stream));
}

// ---------------------------------------------------------------------------
// generic blended evaluation
// ---------------------------------------------------------------------------
namespace {


__device__ int find_cell(const int32_t* cells, int ncell, int cx, int cy, int cz) {
  int lo = 0, hi = ncell - 1;
  while (lo <= hi) {
    const int mid = (lo + hi) >> 1;
    const int* c = cells + 3 * mid;
    int cmp = (c[0] != cx) ? (c[0] < cx ? -1 : 1) : (c[1] != cy) ? (c[1] < cy ? -1 : 1) : (c[2] != cz) ? (c[2] < cz ? -1 : 1) : 0;
    if (cmp == 0) return mid;
    if (cmp < 0) lo = mid + 1; else hi = mid - 1;
  }
  return -1;
}

__device__ __forceinline__ long long floor_div(double v, double s) { return (long long)floor(v / s); }

// Per point and pass: the pass-th candidate expert (in sid order) owning the
// tag's net with a positive gate weight (partition.py:180-229 keeps w > 0).
__global__ void k_pass_keys(int src_kind, const void* src, const int64_t* gather, int64_t n, int pass, const int32_t* cells, int ncell,
                            const int32_t* tagnet, int tag, int S, int halo, uint8_t* ncand, uint16_t* keys,
                            int64_t* vals, BlendOut o, int nokey, int32_t* maxc, const int64_t* n_dev,
                            int32_t* hist, uint8_t* flags, uint16_t* cand) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (n_dev && i >= *n_dev) {  // capacity tail beyond the device count: no candidate, no output
    if (pass == 0) ncand[i] = 0;
    keys[i] = (uint16_t)nokey;
    vals[i] = i;
    if (flags) flags[i] = 0;
    return;
  }
  double c[3];
  point_centre(src_kind, src, gather ? gather[i] : i, c);
  const double h = (double)halo;
  long long lo[3], hi[3];
  for (int a = 0; a < 3; ++a) {
    lo[a] = floor_div(c[a] - h, (double)S);
    hi[a] = floor_div(c[a] + h, (double)S);
  }
  int found = 0;
  int key = nokey;
  for (int combo = 0; combo < 8; ++combo) {
    bool ok = true;
    int cell[3];
    for (int a = 0; a < 3; ++a) {
      const int bit = 4 >> a;
      if (combo & bit) {
        ok &= hi[a] != lo[a];
        cell[a] = (int)hi[a];
      } else {
        cell[a] = (int)lo[a];
      }
    }
    if (!ok) continue;
    const int e = find_cell(cells, ncell, cell[0], cell[1], cell[2]);
    if (e < 0) continue;
    const int net = tagnet[4 * e + tag];
    if (net < 0) continue;
    if (!(gate_weight(cell, S, halo, c, 0.5 / (double)halo) > 0.0)) continue;
    if (found == pass) key = net;
    if (cand) cand[8 * i + found] = (uint16_t)net;  // pass 0 records every candidate for the later passes
    ++found;
  }
  if (pass == 0) {
    ncand[i] = (uint8_t)found;
    if (found > 1) {
      atomicMax(maxc, found);
      atomicAdd(hist + found, 1);  // points with > 1 candidate (the later passes' sizes)
    }
    if (found == 0) {  // uncovered everywhere (inference.py:53-56 -> background)
      switch (o.out_mode) {
        case OUT_PROBS: {
          const int k = (tag == NVDB_TAG_L1) ? 3 : 1;
          for (int j = 0; j < k; ++j) o.out_probs[i * k + j] = 0.0;
          o.out_u8[i] = 0;
          break;
        }
        case OUT_L1CLASS: o.out_u8[i] = 2; break;
        case OUT_L0ACTIVE: o.out_u8[i] = 0; break;
        case OUT_VALUE: o.out_f32[i] = o.background; break;
        default: {
          const int k = (tag == NVDB_TAG_L1) ? 3 : 1;
          for (int j = 0; j < k; ++j) o.out_raw[i * k + j] = 0.f;
          break;
        }
      }
    }
  }
  keys[i] = (uint16_t)key;
  vals[i] = i;
  if (flags) flags[i] = key != nokey ? 1 : 0;
}

// Segments of equal key in the sorted list -> tiles (pairs share a net).
// Tiles of one pass, built in parallel from the net-sorted keys: per net the
// run [start, end) of its points (sentinel keys sort last), ceil(len / 128)
// tiles rounded up to an even count (tiles are launched in pairs).
__global__ void k_run_bounds(const uint16_t* __restrict__ keys, int64_t n, int nokey, int64_t* __restrict__ start,
                             int64_t* __restrict__ end) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint16_t k = keys[i];
  if (k == nokey) return;
  if (i == 0 || keys[i - 1] != k) start[k] = i;
  if (i == n - 1 || keys[i + 1] != k) end[k] = i + 1;
}

__global__ void k_tile_plan(const int64_t* __restrict__ start, const int64_t* __restrict__ end, int nnets,
                            int64_t max_tiles, int64_t* __restrict__ toff, int32_t* __restrict__ npairs) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  int64_t nt = 0;
  for (int k = 0; k < nnets; ++k) {
    toff[k] = nt;
    const int64_t len = end[k] - start[k];
    int64_t cnt = (len + kTileM - 1) / kTileM;
    cnt = (cnt + 1) & ~1LL;
    nt = (nt + cnt < (max_tiles & ~1LL)) ? nt + cnt : (max_tiles & ~1LL);
  }
  toff[nnets] = nt;
  *npairs = (int32_t)(nt / 2);
}

__global__ void k_write_tiles(const int64_t* __restrict__ start, const int64_t* __restrict__ end,
                              const int64_t* __restrict__ toff, int nnets, Tile* __restrict__ tiles) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= toff[nnets]) return;
  int k = 0;
  while (k + 1 < nnets && toff[k + 1] <= t) ++k;
  const int64_t i = t - toff[k];
  const int64_t len = end[k] - start[k];
  const int64_t rem = len - i * kTileM;
  Tile tl;
  tl.net = k;
  tl.first = start[k] + i * kTileM;
  tl.count = (int32_t)(rem < 0 ? 0 : (rem > kTileM ? kTileM : rem));
  tl.flags = 0;
  tl.pad = 0;
  tiles[t] = tl;
}

// keys of a later pass from the candidates pass 0 recorded (no centre /
// cell / gate recomputation): the pass-th candidate's net, or the sentinel
__global__ void k_pass_keys_later(int64_t n, int pass, const uint8_t* __restrict__ ncand,
                                  const uint16_t* __restrict__ cand, int nokey, uint16_t* keys, int64_t* vals,
                                  uint8_t* flags) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const bool has = ncand[i] > pass;
  keys[i] = has ? cand[8 * i + pass] : (uint16_t)nokey;
  vals[i] = i;
  if (flags) flags[i] = has ? 1 : 0;
}

struct WsLayout {
  size_t ncand, keys_in, keys_out, vals_in, vals_out, tiles, npairs, runs, acc, cub, total;
  size_t flags, keys_c, vals_c, nsel, cand;
  size_t cub_bytes;
  int64_t max_tiles;
};

WsLayout ws_layout(const nvdb_netset* ns, int64_t n) {
  WsLayout w{};
  size_t off = 0;
  auto take = [&](size_t b) {
    size_t o = off;
    off = align_up(off + b, 256);
    return o;
  };
  w.max_tiles = n / kTileM + 2 * (int64_t)std::max(ns->nnets, 1) + 4;
  w.ncand = take(n);
  w.keys_in = take(2 * n);
  w.keys_out = take(2 * n);
  w.vals_in = take(8 * n);
  w.vals_out = take(8 * n);
  w.tiles = take(sizeof(Tile) * w.max_tiles);
  w.npairs = take(64);  // npairs | max candidates per point | histogram of candidate counts [9]
  w.flags = take(n);     // later passes: the points that have a candidate in the pass
  w.keys_c = take(2 * n);
  w.vals_c = take(8 * n);
  w.nsel = take(16);
  w.cand = take(16 * n);  // up to 8 candidate nets per point (pass 0)
  w.runs = take(8 * (3 * (size_t)std::max(ns->nnets, 1) + 1));  // start | end | toff (+1)
  w.acc = take(32 * n);
  size_t cub_bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, cub_bytes, (uint16_t*)nullptr, (uint16_t*)nullptr, (int64_t*)nullptr,
                                  (int64_t*)nullptr, (int)std::max<int64_t>(n, 1), 0, 16);
  size_t sel_k = 0, sel_v = 0;
  cub::DeviceSelect::Flagged(nullptr, sel_k, (uint16_t*)nullptr, (uint8_t*)nullptr, (uint16_t*)nullptr, (int*)nullptr,
                             (int)std::max<int64_t>(n, 1));
  cub::DeviceSelect::Flagged(nullptr, sel_v, (int64_t*)nullptr, (uint8_t*)nullptr, (int64_t*)nullptr, (int*)nullptr,
                             (int)std::max<int64_t>(n, 1));
  cub_bytes = std::max(cub_bytes, std::max(sel_k, sel_v));
  w.cub_bytes = cub_bytes;
  w.cub = take(cub_bytes);
  w.total = off;
  return w;
}

}  // namespace

namespace nvdb {

// calls above 2^30 points run in chunks of 2^30 (run_blended): the workspace covers one chunk
size_t blended_workspace_bytes(const nvdb_netset* ns, int64_t n) {
  return ws_layout(ns, std::min<int64_t>(n, int64_t(1) << 30)).total;
}

static int run_blended_one(const nvdb_netset* ns, int tag, int src_kind, const void* src, const int64_t* gather,
                           int64_t n, const BlendOut& o, void* ws, size_t ws_bytes, cudaStream_t st,
                           const int64_t* n_dev) {
  if (n <= 0) return NVDB_OK;
  MlpArgs a{};
  a.src_kind = src_kind;
  a.src = src;
  a.gather = gather;
  a.out_raw = o.out_raw;
  a.out_mode = o.out_mode;
  a.out_probs = o.out_probs;
  a.out_u8 = o.out_u8;
  a.out_f32 = o.out_f32;
  a.value_scale = o.value_scale;
  a.background = o.background;
  a.clip = o.clip;
  // fast path: a single expert needs no dispatch (every point has it as its
  // only candidate; its gate weight decides coverage in the epilogue)
  if (ns->nexperts == 1 && ns->tagnet[tag] >= 0) {
    a.tiles = nullptr;
    a.implicit_net = ns->tagnet[tag];
    a.n_implicit = n;
    a.n_dev = n_dev;
    const int64_t ntiles = (n + kTileM - 1) / kTileM;
    a.npairs = (int32_t)((ntiles + 1) / 2);
    return launch_mlp(ns, a, nullptr, (int)std::min<int64_t>(a.npairs, num_sms()), st);
  }
  const WsLayout w = ws_layout(ns, n);
  if (!ws || ws_bytes < w.total) return fail(NVDB_ENOMEM, "blended workspace %zu < %zu", ws_bytes, w.total);
  uint8_t* base = static_cast<uint8_t*>(ws);
  uint8_t* ncand = base + w.ncand;
  uint16_t* kin = reinterpret_cast<uint16_t*>(base + w.keys_in);
  uint16_t* kout = reinterpret_cast<uint16_t*>(base + w.keys_out);
  int64_t* vin = reinterpret_cast<int64_t*>(base + w.vals_in);
  int64_t* vout = reinterpret_cast<int64_t*>(base + w.vals_out);
  Tile* tiles = reinterpret_cast<Tile*>(base + w.tiles);
  int32_t* npairs = reinterpret_cast<int32_t*>(base + w.npairs);
  a.acc = reinterpret_cast<double*>(base + w.acc);
  a.ncand = ncand;
  a.tiles = tiles;
  a.idx = vout;
  const int threads = 256;
  const int blocks = (int)((n + threads - 1) / threads);
  // sentinel key = nnets sorts last; radix digits only over the bits a net index needs
  const int nokey = ns->nnets;
  int kbits = 1;
  while ((1 << kbits) <= nokey) ++kbits;
  int32_t* maxc = npairs + 1;
  int32_t* hist = npairs + 2;  // [9]
  uint8_t* flags = base + w.flags;
  uint16_t* kc = reinterpret_cast<uint16_t*>(base + w.keys_c);
  int64_t* vc = reinterpret_cast<int64_t*>(base + w.vals_c);
  int* nsel = reinterpret_cast<int*>(base + w.nsel);
  uint16_t* cand = reinterpret_cast<uint16_t*>(base + w.cand);
  int passes = 8;
  int32_t hh[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};  // maxc | hist[0..8]
  for (int pass = 0; pass < passes; ++pass) {
    // pass 0 sorts every point; a later pass p only the points with more than
    // p candidates (counted in pass 0), compacted first in their original
    // order -- the same subsequence the full stable sort would put before
    // the sentinel keys, so the tiles and results are unchanged
    int64_t np_ = n;
    if (pass > 0) {
      np_ = 0;
      for (int c = pass + 1; c <= 8; ++c) np_ += hh[1 + c];
      if (np_ == 0) continue;
    }
    const bool compact = pass > 0 && np_ < n;
    if (pass == 0) NVDB_CUDA_TRY(cudaMemsetAsync(maxc, 0, 40, st));
    if (pass == 0) {
      k_pass_keys<<<blocks, threads, 0, st>>>(src_kind, src, gather, n, pass, ns->dev_cells, ns->nexperts,
                                              ns->dev_tagnet, tag, ns->subdomain_size, ns->halo, ncand, kin, vin, o,
                                              nokey, maxc, n_dev, hist, nullptr, cand);
    } else {
      k_pass_keys_later<<<blocks, threads, 0, st>>>(n, pass, ncand, cand, nokey, kin, vin, compact ? flags : nullptr);
    }
    NVDB_CHECK_LAUNCH();
    if (pass == 0) {  // later passes only exist up to the largest candidate count of this call
      NVDB_CUDA_TRY(cudaMemcpyAsync(hh, maxc, 40, cudaMemcpyDeviceToHost, st));
      NVDB_CUDA_TRY(cudaStreamSynchronize(st));
      passes = std::max(1, std::min(8, (int)hh[0]));
    }
    const uint16_t* ksrc = kin;
    const int64_t* vsrc = vin;
    if (compact) {
      size_t cs = w.cub_bytes;
      NVDB_CUDA_TRY(cub::DeviceSelect::Flagged(base + w.cub, cs, kin, flags, kc, nsel, (int)n, st));
      cs = w.cub_bytes;
      NVDB_CUDA_TRY(cub::DeviceSelect::Flagged(base + w.cub, cs, vin, flags, vc, nsel, (int)n, st));
      ksrc = kc;
      vsrc = vc;
    }
    size_t cb = w.cub_bytes;
    NVDB_CUDA_TRY(cub::DeviceRadixSort::SortPairs(base + w.cub, cb, ksrc, kout, vsrc, vout, (int)np_, 0, kbits, st));
    {
      const int nn = std::max(ns->nnets, 1);
      int64_t* rs = reinterpret_cast<int64_t*>(base + w.runs);
      int64_t* re = rs + nn;
      int64_t* to = re + nn;
      NVDB_CUDA_TRY(cudaMemsetAsync(rs, 0, 16 * (size_t)nn, st));
      k_run_bounds<<<(int)((np_ + threads - 1) / threads), threads, 0, st>>>(kout, np_, nokey, rs, re);
      NVDB_CHECK_LAUNCH();
      k_tile_plan<<<1, 32, 0, st>>>(rs, re, ns->nnets, w.max_tiles, to, npairs);
      NVDB_CHECK_LAUNCH();
      k_write_tiles<<<(int)((w.max_tiles + 255) / 256), 256, 0, st>>>(rs, re, to, ns->nnets, tiles);
      NVDB_CHECK_LAUNCH();
    }
    a.pass = pass;
    int rc = launch_mlp(ns, a, npairs, num_sms(), st);
    if (rc) return rc;
  }
  return NVDB_OK;
}

// Calls above 2^30 points run as consecutive chunks of 2^30 (a multiple of
// the 4096 points of a level-1 node, so implicit leaf-voxel / slot ids keep
// their node): the tile indices, radix sorts and selections inside one
// chunk stay in 32-bit range.  A chunk's source, gather list and outputs are
// the caller's arrays advanced to its first point; the workspace sized for n
// covers any chunk.  A device-held count (n_dev) cannot be split on the host.
int run_blended(const nvdb_netset* ns, int tag, int src_kind, const void* src, const int64_t* gather, int64_t n,
                const BlendOut& o, void* ws, size_t ws_bytes, cudaStream_t st, const int64_t* n_dev) {
  constexpr int64_t kChunk = int64_t(1) << 30;
  if (n <= kChunk) return run_blended_one(ns, tag, src_kind, src, gather, n, o, ws, ws_bytes, st, n_dev);
  if (n_dev) return fail(NVDB_EUNSUPPORTED, "run_blended: a device-counted call above 2^30 points");
  int out_dim = 1;
  for (int e = 0; e < ns->nexperts; ++e) {
    const int ni = ns->tagnet[e * 4 + tag];
    if (ni >= 0) {
      out_dim = ns->nets[ni].out_dim;
      break;
    }
  }
  for (int64_t s0 = 0; s0 < n; s0 += kChunk) {
    const int64_t m = std::min(kChunk, n - s0);
    const void* csrc = src;
    const int64_t* cg = gather;
    if (gather) {
      cg = gather + s0;
    } else {
      switch (src_kind) {
        case SRC_NORM_F32: csrc = static_cast<const float*>(src) + 3 * s0; break;
        case SRC_CENTER_F64: csrc = static_cast<const double*>(src) + 3 * s0; break;
        case SRC_COORD_I32: csrc = static_cast<const int32_t*>(src) + 3 * s0; break;
        case SRC_LEAF_VOX: csrc = static_cast<const int32_t*>(src) + 3 * (s0 >> 9); break;
        case SRC_L1_SLOT: csrc = static_cast<const int32_t*>(src) + 3 * (s0 >> 12); break;
        default: return fail(NVDB_EINVAL, "run_blended: bad source kind %d", src_kind);
      }
    }
    BlendOut c = o;
    if (c.out_raw) c.out_raw += s0 * out_dim;
    if (c.out_probs) c.out_probs += s0 * out_dim;
    if (c.out_u8) c.out_u8 += s0;
    if (c.out_f32) c.out_f32 += s0;
    const int rc = run_blended_one(ns, tag, src_kind, csrc, cg, m, c, ws, ws_bytes, st, nullptr);
    if (rc) return rc;
  }
  return NVDB_OK;
}

}  // namespace nvdb

extern "C" size_t nvdb_eval_workspace_bytes(const nvdb_netset* ns, int64_t n) {
  return ns ? blended_workspace_bytes(ns, n) : 0;
}

extern "C" int nvdb_eval_blended(const nvdb_netset* ns, int32_t tag, const double* centers, int64_t n, double* out,
                                 uint8_t* covered, void* workspace, size_t workspace_bytes, void* stream) {
  if (!ns || tag < 0 || tag > 3) return fail(NVDB_EINVAL, "nvdb_eval_blended: bad netset/tag");
  if (n < 0 || (n > 0 && (!centers || !out || !covered))) return fail(NVDB_EINVAL, "nvdb_eval_blended: bad buffers");
  BlendOut o{};
  o.out_mode = OUT_PROBS;
  o.out_probs = out;
  o.out_u8 = covered;
  return run_blended(ns, tag, SRC_CENTER_F64, centers, nullptr, n, o, workspace, workspace_bytes,
                     static_cast<cudaStream_t>(stream));
}

// ---------------------------------------------------------------------------
// descriptor self-test: one 128xN MMA from caller-laid-out smem images
// ---------------------------------------------------------------------------
namespace {

__global__ void k_selftest_umma(const uint8_t* a_img, uint32_t a_bytes, const uint8_t* b_img, uint32_t b_bytes,
                                int n, int nk, uint32_t a_lbo, uint32_t a_sbo, uint32_t a_step, uint32_t b_lbo,
                                uint32_t b_sbo, uint32_t b_step, int a_mn, int b_mn, float* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  uint8_t* sa = sm;
  uint8_t* sb = sm + ((a_bytes + 1023u) & ~1023u);
  for (uint32_t i = threadIdx.x; i < a_bytes; i += blockDim.x) sa[i] = a_img[i];
  for (uint32_t i = threadIdx.x; i < b_bytes; i += blockDim.x) sb[i] = b_img[i];
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (threadIdx.x < 32) tmem_alloc(&tslot, 512);
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tslot;
  const bool a_tmem = (a_mn == 2);  // A (row-major 128 x K fp16) staged in TMEM columns 256..
  if (a_tmem) {
    const int row = threadIdx.x;
    const uint32_t* arow = reinterpret_cast<const uint32_t*>(sa) + row * (nk * 8);
    for (int c = 0; c < nk * 8; c += 8) {
      uint32_t r[8];
      for (int i = 0; i < 8; ++i) r[i] = arow[c + i];
      tmem_st8(tm + 256 + c + ((uint32_t)((threadIdx.x >> 5) * 32) << 16), r);
    }
    tmem_st_wait();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
  }
  if (threadIdx.x == 0) {
    const uint32_t idesc = idesc_f16(128, n, a_tmem ? 0 : a_mn, b_mn);
    for (int s = 0; s < nk; ++s) {
      const uint64_t bd = smem_desc(smem_addr(sb) + s * b_step, b_lbo, b_sbo);
      if (a_tmem) {
        umma_f16_ts(tm, tm + 256 + s * 8, bd, idesc, s != 0);
      } else {
        const uint64_t ad = smem_desc(smem_addr(sa) + s * a_step, a_lbo, a_sbo);
        umma_f16(tm, ad, bd, idesc, s != 0);
      }
    }
    umma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  const int warp = threadIdx.x >> 5;
  const int row = threadIdx.x;
  for (int c = 0; c < n; c += 16) {
    float v[16];
    tmem_ld16(tm + ((uint32_t)(warp * 32) << 16) + c, v);
    tmem_ld_wait();
    for (int i = 0; i < 16; ++i) out[row * n + c + i] = v[i];
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(tm, 512);
}

}  // namespace

extern "C" int nvdb_selftest_umma(const void* a_img, uint32_t a_bytes, const void* b_img, uint32_t b_bytes, int32_t n,
                                  int32_t nk, uint32_t a_lbo, uint32_t a_sbo, uint32_t a_step, uint32_t b_lbo,
                                  uint32_t b_sbo, uint32_t b_step, int32_t a_mn, int32_t b_mn, float* out,
                                  void* stream) {
  if (n < 16 || n > 256 || n % 16 || nk < 1) return fail(NVDB_EINVAL, "selftest: bad n/nk");
  const uint32_t smem = (uint32_t)(align_up(a_bytes, 1024) + align_up(b_bytes, 1024));
  if (smem > kMaxDynSmem) return fail(NVDB_EINVAL, "selftest: images too large");
  if (enable_max_smem(k_selftest_umma) < (long long)smem) return fail(NVDB_ECUDA, "selftest: smem limit");
  k_selftest_umma<<<1, 128, smem, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const uint8_t*>(a_img), a_bytes, static_cast<const uint8_t*>(b_img), b_bytes, n, nk, a_lbo, a_sbo,
      a_step, b_lbo, b_sbo, b_step, a_mn, b_mn, out);
  NVDB_CHECK_LAUNCH();
  return NVDB_OK;
}
