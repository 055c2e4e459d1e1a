// Layer-streamed training of wide coordinate networks (Table-3 shapes:
// hidden width up to 256, 2m up to 1024), one epoch of neural.fused_step
// (neural.py:444-524) in two kernels, used when the net's weights or its
// per-tile backward state do not fit the fused narrow kernels of train.cu:
//
//   k_lw_fb   per 128-sample tile, one tile per 4-warp engine: gather, Fourier
//             features, forward on tcgen05 (one W-column fp32 accumulator in
//             TMEM per engine), fp32 head, loss and dL/dout, then the dgrad
//             chain back to layer 0.  Weights are not resident: the net's
//             fp16 image [W_0 | W_1 .. W_{d-1} | W_{d-1}^T .. W_1^T] is consumed
//             as its sequence of K = 16 chunks (W x 32 bytes) through a ring
//             of bulk async copies shared by the CTA's engines (a chunk fetched
//             from L2 serves every engine's current tile).  The transposed
//             copies make the dgrad B operand the same K-major chunk as the
//             forward one.  Features, activations, f'(z) and dz go to fp16
//             tile images in global memory for the weight gradients; f'(z) of
//             the lower layers is read back in the backward pass (the top
//             layer's is recomputed from its accumulator, still in TMEM).
//   k_lw_wg   weight gradients as split-K tcgen05 GEMMs over the tile images:
//             work item = (128-row block of one layer's inputs, sample split);
//             D[in, out] += A^T dz with A (features / activations) and dz read
//             MN-major from the same K-major images; bias gradients of the
//             layer's out-block from dz x ones in the same pass; fixed
//             split boundaries, per-split partials reduced in a fixed order by
//             k_train_adam (bitwise-deterministic).
//
// Scaling conventions are the narrow path's: the fp16 images carry omega (and
// the feature amplitude) folded in, f'(z) = d act / d z' without omega, and
// dL/dout without 1/size; k_train_adam applies 1/size and omega in fp32.
#pragma once

constexpr int kLwMaxEngines = 4;
constexpr int kLwRing = 8;             // weight ring slots (W x 32 bytes each)
constexpr int kLwChunkK = 64;          // feature K per chunk (4 MMAs of K = 16)
constexpr int kLwChunkBytes = kTileM * kLwChunkK * 2;  // 16 KB

struct LwPlan {
  int engines = 0;
  uint32_t ereg = 0;       // bytes per engine: 2 feature slots / the fp16 A tile (activations, dz)
  uint32_t ring_off = 0, small_off = 0, bar_off = 0, total = 0;
  int sm_bias = 0, sm_headw = 0, sm_headb = 0, sm_b2pi = 0, sm_loss = 0;
};

inline LwPlan plan_lw(int W, int depth, int k0, uint32_t limit) {
  LwPlan p;
  auto a4 = [](int v) { return (v + 3) & ~3; };
  p.sm_bias = 0;
  p.sm_headw = a4(depth * W);
  p.sm_headb = p.sm_headw + a4(3 * W);
  p.sm_b2pi = p.sm_headb + 4;
  p.sm_loss = p.sm_b2pi + a4(3 * (k0 / 2));
  const uint32_t small_bytes = (uint32_t)(p.sm_loss + 2 * kLwMaxEngines * 4) * 4u;  // + loss scratch (double)
  p.ereg = (uint32_t)align_up(std::max<size_t>((size_t)2 * kLwChunkBytes, (size_t)kTileM * W * 2), 1024);
  const uint32_t ring_bytes = (uint32_t)kLwRing * (uint32_t)W * 32u;
  const int by_tmem = std::min(kLwMaxEngines, 512 / W);
  for (int e = by_tmem; e >= 1; --e) {
    const uint32_t tot = (uint32_t)e * p.ereg + ring_bytes + (uint32_t)align_up(small_bytes, 16) + 512;
    if (tot <= limit) {
      p.engines = e;
      break;
    }
  }
  p.ring_off = (uint32_t)p.engines * p.ereg;
  p.small_off = p.ring_off + ring_bytes;
  p.bar_off = (uint32_t)align_up(p.small_off + small_bytes, 16);
  p.total = p.bar_off + 512;  // 32 mbarriers + the TMEM address slot
  return p;
}

struct LwFbArgs {
  NetDev net;                 // wimg = [forward | transposed] image, bias' (omega b), head, b2pi
  uint32_t nk_fwd, nk_tot;    // K = 16 chunks of the forward part / of the whole image
  const float* xs;
  const float* ys;
  const int64_t* idx;
  const int32_t* idx_all;
  const int32_t* epoch;
  int64_t batch;
  int64_t tile_begin, tile_end;
  int32_t loss_kind;
  uint16_t* feat_img;         // [ntiles][128 x k0]
  uint16_t* act_img;          // [depth][ntiles][128 x W]
  uint16_t* fp_img;           // [depth - 1][ntiles][128 x W] f'(z) of the lower layers
  uint16_t* dz_img;           // [depth][ntiles][128 x W]
  uint16_t* dlt_img;          // [ntiles][128 x 16]
  double* loss_part;          // [grid]
  const int32_t* stopped;
  LwPlan plan;
};

__global__ void __launch_bounds__(128 * kLwMaxEngines, 1) k_lw_fb(const LwFbArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  if (*a.stopped) return;
  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int g = tid >> 7;   // engine
  const int p = tid & 127;  // tile row == TMEM lane
  const int E = a.plan.engines;
  const int nthreads = 128 * E;
  const NetDev& nd = a.net;
  const int W = nd.width, depth = nd.depth, k0 = nd.k0, out_dim = nd.out_dim, act = nd.act;
  const int mp = k0 >> 1;
  float* small = reinterpret_cast<float*>(smem + a.plan.small_off);
  float* s_bias = small + a.plan.sm_bias;
  float* s_headw = small + a.plan.sm_headw;
  float* s_headb = small + a.plan.sm_headb;
  float* s_b2pi = small + a.plan.sm_b2pi;
  double* s_loss = reinterpret_cast<double*>(small + a.plan.sm_loss);  // [engines][4] warp partials
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + a.plan.bar_off);
  uint64_t* slot_free = bars + 4 * g;  // [2] feature slot free (MMA commit)
  uint64_t* mdone = slot_free + 2;     // layer MMAs complete
  uint64_t* wfull = bars + 16;         // [kLwRing]
  uint64_t* wempty = wfull + kLwRing;  // [kLwRing], count E
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(wempty + kLwRing);
  __shared__ uint32_t s_wnext;

  if (tid == 0) {
    for (int e = 0; e < E; ++e)
      for (int s = 0; s < 3; ++s) mbar_init(bars + 4 * e + s, 1);
    for (int s = 0; s < kLwRing; ++s) {
      mbar_init(wfull + s, 1);
      mbar_init(wempty + s, E);
    }
    s_wnext = 0;
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(tmem_slot, 512);
  for (int i = tid; i < depth * W; i += nthreads) s_bias[i] = nd.bias[i];
  for (int i = tid; i < out_dim * W; i += nthreads) s_headw[i] = nd.headw[i];
  if (tid < out_dim) s_headb[tid] = nd.headb[tid];
  for (int i = tid; i < 3 * mp; i += nthreads) s_b2pi[i] = nd.b2pi[i];
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const uint32_t zcol = tmem_base + (uint32_t)(g * W);
  const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
  const uint32_t region = smem_addr(smem) + (uint32_t)g * a.plan.ereg;  // feature slots / A tile
  const bool issuer = p == 0;
  const uint32_t idesc = idesc_f16(kTileM, W, 0, 0);
  const uint32_t cb = (uint32_t)W * 32u;  // bytes per weight chunk
  const uint32_t ring_s = smem_addr(smem + a.plan.ring_off);
  uint8_t* const ring_p = smem + a.plan.ring_off;
  const uint32_t nk = a.nk_tot;

  // ---- weight ring (issuer threads): slots of wp consecutive chunks (one
  // bulk copy, one barrier round and one commit per slot: the issuer's
  // per-slot bookkeeping costs several MMAs' worth of clocks, see
  // mlp_eval_kernel), kLwRing / wp slots; positions count up over the whole
  // launch, slot chunk group c = pos % (nk / wp); any engine's issuer may
  // claim the next position; a slot is refilled once every engine consumed it
  uint32_t wp = 1;
  {
    uint32_t g0 = (uint32_t)k0 / 16u, h0 = (uint32_t)W / 16u;
    while (h0) {
      const uint32_t r = g0 % h0;
      g0 = h0;
      h0 = r;
    }
    for (uint32_t q = 4; q > 1; q >>= 1)
      if (g0 % q == 0 && nk % q == 0) {
        wp = q;
        break;
      }
  }
  const uint32_t WRn = (uint32_t)kLwRing / wp, sb = cb * wp, nkp = nk / wp;
  const uint32_t wslack = WRn >= 3 ? 1u : 0u;
  const uint32_t wdstep = (uint32_t)W * 2u;  // one chunk in descriptor units (W x 32 bytes >> 4)
  uint32_t wcons = 0, wcur = 0, wph = 0, wpc = 0;
  uint64_t wdesc = 0;
  auto w_fill_pos = [&](uint32_t pos) {
    const uint32_t slot = pos % WRn;
    if (pos >= WRn) mbar_wait(wempty + slot, ((pos / WRn) - 1) & 1u);
    mbar_arrive_expect_tx(wfull + slot, sb);
    bulk_g2s(ring_p + slot * sb, nd.wimg + (size_t)(pos % nkp) * sb, sb, wfull + slot);
  };
  auto w_refill = [&]() {  // prefetch into slots that are already free
    while (true) {
      const uint32_t n = *reinterpret_cast<volatile uint32_t*>(&s_wnext);
      if (n >= wcons + WRn - wslack) break;
      if (n >= WRn && !mbar_test(wempty + n % WRn, ((n / WRn) - 1) & 1u)) break;
      if (atomicCAS(&s_wnext, n, n + 1) == n) w_fill_pos(n);
    }
  };
  auto w_next = [&]() {
    w_refill();
    while (true) {  // this issuer's own position must be claimed (blocking only for it)
      const uint32_t n = *reinterpret_cast<volatile uint32_t*>(&s_wnext);
      if (n > wcons) break;
      if (atomicCAS(&s_wnext, n, n + 1) == n) w_fill_pos(n);
    }
    mbar_wait(wfull + wcur, wph);
    wdesc = smem_desc(ring_s + wcur * sb, W * 16, 128);
  };
  auto w_advance = [&]() {
    ++wcons;
    if (++wcur == WRn) {
      wcur = 0;
      wph ^= 1u;
    }
  };
  auto w_mma = [&](uint64_t adesc, uint32_t acc) {
    if (wpc == 0) w_next();
    umma_f16(zcol, adesc, wdesc + (uint64_t)(wpc * wdstep), idesc, acc);
    if (++wpc == wp) {
      umma_commit(wempty + wcur);
      w_advance();
      wpc = 0;
      w_refill();
    }
  };
  // `cnt` consecutive chunks (A advancing 256 = 4 KB per step): whole
  // 4-chunk slots go out as one umma_f16_x4 (one ELECT/R2UR sequence)
  auto w_mma_run = [&](uint64_t adesc, uint32_t acc, int cnt) {
    for (int k = 0; k < cnt;) {
      if (wpc == 0 && wp == 4 && cnt - k >= 4) {
        w_next();
        umma_f16_x4(zcol, adesc, wdesc, idesc, acc, 256, wdstep);
        umma_commit(wempty + wcur);
        w_advance();
        w_refill();
        k += 4;
        adesc += 1024;
      } else {
        w_mma(adesc, acc);
        ++k;
        adesc += 256;
      }
      acc = 1;
    }
  };
  auto w_skip_tile = [&]() {
    for (uint32_t c = 0; c < nkp; ++c) {
      w_next();
      mbar_arrive(wempty + wcur);
      w_advance();
    }
  };

  const int64_t ntiles = (a.batch + kTileM - 1) / kTileM;
  const int64_t per = (a.tile_end - a.tile_begin + gridDim.x - 1) / gridDim.x;
  const int64_t t0 = a.tile_begin + blockIdx.x * per, t1 = min(a.tile_end, t0 + per);
  const int32_t* eidx = a.idx_all ? a.idx_all + (int64_t)(*a.epoch) * a.batch : nullptr;
  const size_t tile_elems = (size_t)kTileM * W;
  uint32_t cc = 0, mpar = 0;
  double loss_acc = 0.0;

  auto process = [&](int64_t tau) {
    const int64_t b = tau * kTileM + p;
    const bool valid = b < a.batch;
    float x0 = 0.f, x1 = 0.f, x2 = 0.f, y = 0.f;
    if (valid) {
      const int64_t pi = eidx ? (int64_t)eidx[b] : (a.idx ? a.idx[b] : b);
      x0 = a.xs[3 * pi]; x1 = a.xs[3 * pi + 1]; x2 = a.xs[3 * pi + 2];
      y = a.ys[pi];
    }
    // ---------------- features -> layer 0 (K chunks of 64)
    uint8_t* gfeat = reinterpret_cast<uint8_t*>(a.feat_img) + (size_t)tau * kTileM * k0 * 2;
    const int nch = k0 / kLwChunkK;
    for (int ch = 0; ch < nch; ++ch, ++cc) {
      const uint32_t s = cc & 1u;
      if (cc >= 2) mbar_wait(slot_free + s, ((cc >> 1) - 1) & 1u);
      const uint32_t buf = region + s * kLwChunkBytes;
#pragma unroll 2
      for (int q = 0; q < kLwChunkK / 8; ++q) {
        const int f0 = ch * (kLwChunkK / 2) + q * 4;
        const float4 bx = *reinterpret_cast<const float4*>(s_b2pi + f0);
        const float4 by = *reinterpret_cast<const float4*>(s_b2pi + mp + f0);
        const float4 bz = *reinterpret_cast<const float4*>(s_b2pi + 2 * mp + f0);
        const float bxa[4] = {bx.x, bx.y, bx.z, bx.w}, bya[4] = {by.x, by.y, by.z, by.w};
        const float bza[4] = {bz.x, bz.y, bz.z, bz.w};
        uint32_t h[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float th = fmaf(x2, bza[j], fmaf(x1, bya[j], x0 * bxa[j]));
          float sv, cv;
          __sincosf(th, &sv, &cv);
          h[j] = pack_half2(cv, sv);
        }
        const uint32_t fo = kmajor_offset(p, q * 8, kTileM);
        st_shared_v4(buf + fo, h[0], h[1], h[2], h[3]);
        *reinterpret_cast<uint4*>(gfeat + (size_t)ch * kLwChunkBytes + fo) = make_uint4(h[0], h[1], h[2], h[3]);
      }
      fence_async_smem();
      tc_fence_before();
      named_bar_sync(1 + g, 128);
      if (issuer) {
        tc_fence_after();
        const uint64_t ad = smem_desc(buf, kTileM * 16, 128);
#pragma unroll
        w_mma_run(ad, ch != 0 ? 1u : 0u, kLwChunkK / 16);
        umma_commit(slot_free + s);
        if (ch == nch - 1) umma_commit(mdone);
      }
    }
    // ---------------- hidden layers (forward)
    float yv[3] = {0.f, 0.f, 0.f};
    for (int l = 0; l < depth; ++l) {
      const bool last = l == depth - 1;
      mbar_wait(mdone, mpar);
      mpar ^= 1u;
      tc_fence_after();
      const float* bl = s_bias + l * W;
      uint8_t* gact = reinterpret_cast<uint8_t*>(a.act_img + ((size_t)l * ntiles + tau) * tile_elems);
      uint8_t* gfp = last ? nullptr : reinterpret_cast<uint8_t*>(a.fp_img + ((size_t)l * ntiles + tau) * tile_elems);
      for (int c = 0; c < W / 16; ++c) {
        float v[16];
        tmem_ld16(zcol + lane_off + c * 16, v);
        tmem_ld_wait();
        float av[16], fv[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const float z = v[i] + bl[c * 16 + i];
          av[i] = act_fn(act, z);
          if (!last) fv[i] = act == ACT_SINE ? __cosf(z) : (act == ACT_TANH ? 1.0f - av[i] * av[i] : (z > 0.f ? 1.f : 0.f));
        }
        uint32_t ap[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) ap[i] = pack_half2(av[2 * i], av[2 * i + 1]);
        const uint32_t o0 = kmajor_offset(p, c * 16, kTileM), o1 = o0 + kTileM * 16;
        *reinterpret_cast<uint4*>(gact + o0) = make_uint4(ap[0], ap[1], ap[2], ap[3]);
        *reinterpret_cast<uint4*>(gact + o1) = make_uint4(ap[4], ap[5], ap[6], ap[7]);
        if (!last) {
          st_shared_v4(region + o0, ap[0], ap[1], ap[2], ap[3]);
          st_shared_v4(region + o1, ap[4], ap[5], ap[6], ap[7]);
          uint32_t fp[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) fp[i] = pack_half2(fv[2 * i], fv[2 * i + 1]);
          *reinterpret_cast<uint4*>(gfp + o0) = make_uint4(fp[0], fp[1], fp[2], fp[3]);
          *reinterpret_cast<uint4*>(gfp + o1) = make_uint4(fp[4], fp[5], fp[6], fp[7]);
        } else {
#pragma unroll
          for (int k = 0; k < 3; ++k) {
            if (k < out_dim) {
              const float* hw = s_headw + k * W + c * 16;
              float sp[4];
#pragma unroll
              for (int q4 = 0; q4 < 4; ++q4) {
                sp[q4] = fmaf(av[4 * q4], hw[4 * q4], av[4 * q4 + 1] * hw[4 * q4 + 1]);
                sp[q4] = fmaf(av[4 * q4 + 2], hw[4 * q4 + 2], sp[q4]);
                sp[q4] = fmaf(av[4 * q4 + 3], hw[4 * q4 + 3], sp[q4]);
              }
              yv[k] += (sp[0] + sp[1]) + (sp[2] + sp[3]);
            }
          }
        }
      }
      if (!last) {
        fence_async_smem();
        tc_fence_before();
        named_bar_sync(1 + g, 128);
        if (issuer) {
          tc_fence_after();
          const uint64_t ad = smem_desc(region, kTileM * 16, 128);
          w_mma_run(ad, 0u, W / 16);
          umma_commit(mdone);
        }
      }
    }
    // ---------------- loss and dL/dout (neural.py:271-302, without 1/size)
    float dl[3] = {0.f, 0.f, 0.f};
    float lterm = 0.f;
#pragma unroll
    for (int k = 0; k < 3; ++k)
      if (k < out_dim) yv[k] += s_headb[k];
    if (valid) {
      if (a.loss_kind == 0) {
        const float d = yv[0] - y;
        lterm = d * d;
        dl[0] = 2.0f * d;
      } else if (a.loss_kind == 2) {
        const float z = yv[0];
        lterm = fmaxf(z, 0.f) - z * y + log1pf(expf(-fabsf(z)));
        dl[0] = 1.0f / (1.0f + expf(-z)) - y;
      } else {
        const float zm = fmaxf(fmaxf(yv[0], yv[1]), yv[2]);
        const float e0 = expf(yv[0] - zm), e1 = expf(yv[1] - zm), e2 = expf(yv[2] - zm);
        const float s = (e0 + e1) + e2;
        const int lab = (int)y;
        const float zl = lab == 0 ? yv[0] : (lab == 1 ? yv[1] : yv[2]);
        lterm = -(zl - zm - logf(s));
        dl[0] = e0 / s - (lab == 0 ? 1.f : 0.f);
        dl[1] = e1 / s - (lab == 1 ? 1.f : 0.f);
        dl[2] = e2 / s - (lab == 2 ? 1.f : 0.f);
      }
    }
    {
      uint8_t* gd = reinterpret_cast<uint8_t*>(a.dlt_img + (size_t)tau * kTileM * 16);
      *reinterpret_cast<uint4*>(gd + kmajor_offset(p, 0, kTileM)) =
          make_uint4(pack_half2(dl[0], dl[1]), pack_half2(dl[2], 0.f), 0u, 0u);
      *reinterpret_cast<uint4*>(gd + kmajor_offset(p, 8, kTileM)) = make_uint4(0u, 0u, 0u, 0u);
    }
    // deterministic loss sum: warp shuffle, then the engine's 4 warps in order
    float ls = lterm;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ls += __shfl_xor_sync(0xffffffffu, ls, o);
    if ((p & 31) == 0) s_loss[4 * g + (p >> 5)] = (double)ls;
    // ---------------- backward: top layer from its accumulator (still in TMEM)
    for (int l = depth - 1; l >= 0; --l) {
      const bool top = l == depth - 1;
      if (!top) {
        mbar_wait(mdone, mpar);
        mpar ^= 1u;
        tc_fence_after();
      }
      const float* bl = s_bias + l * W;
      uint8_t* gdz = reinterpret_cast<uint8_t*>(a.dz_img + ((size_t)l * ntiles + tau) * tile_elems);
      const uint8_t* gfp = top ? nullptr : reinterpret_cast<const uint8_t*>(a.fp_img + ((size_t)l * ntiles + tau) * tile_elems);
      for (int c = 0; c < W / 16; ++c) {
        float v[16], da[16], f[16];
        tmem_ld16(zcol + lane_off + c * 16, v);
        tmem_ld_wait();
        const uint32_t o0 = kmajor_offset(p, c * 16, kTileM), o1 = o0 + kTileM * 16;
        if (top) {
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const float z = v[i] + bl[c * 16 + i];
            f[i] = act == ACT_SINE ? __cosf(z) : (act == ACT_TANH ? 1.0f - tanhf(z) * tanhf(z) : (z > 0.f ? 1.f : 0.f));
            float s2 = 0.f;
#pragma unroll
            for (int k = 0; k < 3; ++k)
              if (k < out_dim) s2 = fmaf(dl[k], s_headw[k * W + c * 16 + i], s2);
            da[i] = s2;
          }
        } else {
          const uint4 q0 = *reinterpret_cast<const uint4*>(gfp + o0);
          const uint4 q1 = *reinterpret_cast<const uint4*>(gfp + o1);
          const uint32_t qq[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const float2 ff = __half22float2(*reinterpret_cast<const __half2*>(&qq[i]));
            f[2 * i] = ff.x;
            f[2 * i + 1] = ff.y;
          }
#pragma unroll
          for (int i = 0; i < 16; ++i) da[i] = v[i];
        }
        uint32_t dp[8];
#pragma unroll
        for (int i = 0; i < 8; ++i)
          dp[i] = valid ? pack_half2(da[2 * i] * f[2 * i], da[2 * i + 1] * f[2 * i + 1]) : 0u;
        *reinterpret_cast<uint4*>(gdz + o0) = make_uint4(dp[0], dp[1], dp[2], dp[3]);
        *reinterpret_cast<uint4*>(gdz + o1) = make_uint4(dp[4], dp[5], dp[6], dp[7]);
        if (l > 0) {
          st_shared_v4(region + o0, dp[0], dp[1], dp[2], dp[3]);
          st_shared_v4(region + o1, dp[4], dp[5], dp[6], dp[7]);
        }
      }
      if (l > 0) {  // da_{l-1} = dz_l . (omega W_l): B = the transposed image's chunks
        fence_async_smem();
        tc_fence_before();
        named_bar_sync(1 + g, 128);
        if (issuer) {
          tc_fence_after();
          const uint64_t ad = smem_desc(region, kTileM * 16, 128);
          w_mma_run(ad, 0u, W / 16);
          umma_commit(mdone);
        }
      }
    }
    tc_fence_before();
    named_bar_sync(1 + g, 128);  // TMEM reads of this tile done before the next tile's MMAs; s_loss published
    if (p == 0) loss_acc += ((s_loss[4 * g] + s_loss[4 * g + 1]) + s_loss[4 * g + 2]) + s_loss[4 * g + 3];
  };

  for (int64_t base = t0; base < t1; base += E) {
    const int64_t tau = base + g;
    if (tau < t1) process(tau);
    else if (issuer) w_skip_tile();
  }
  // per-CTA loss partial, engines in order
  __syncthreads();
  if (p == 0) s_loss[4 * g] = loss_acc;
  __syncthreads();
  if (tid == 0) {
    double sl = 0.0;
    for (int e = 0; e < E; ++e) sl += s_loss[4 * e];
    a.loss_part[blockIdx.x] = sl;
    for (uint32_t pos = wcons; pos < s_wnext; ++pos)  // prefetched slots nobody will use
      mbar_wait(wfull + pos % WRn, (pos / WRn) & 1u);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem_base, 512);
}

// ------------------------------------------------------------------ weight gradients
struct LwBlock {
  int32_t layer;     // 0..depth-1: hidden weight W_layer; depth: the head
  int32_t mblk;      // 128-row block of the layer's inputs
  int32_t n;         // accumulator columns: W (hidden) or 16 (head)
  int32_t bias_blk;  // >= 0: bias gradient of out-block bias_blk in the same pass (-1 none)
  int32_t in_real, out_real;
  int32_t a_rows;    // rows of the input block present in the image (<= 128)
  int32_t pad;
  int64_t w_off, b_off;  // parameter offsets of W_layer / b_layer
};

constexpr uint32_t kLwWgStage = 32768 + 65536;  // A block (128 x 128 fp16) + B tile (128 x <= 256 fp16)
constexpr uint32_t kLwWgSmem = 2 * kLwWgStage + 4096 + 256;

struct LwWgArgs {
  const LwBlock* blocks;
  int32_t nblocks, nsplit;
  int32_t W, depth, k0;
  int64_t batch, tile_begin, tile_end;
  const uint16_t* feat_img;
  const uint16_t* act_img;
  const uint16_t* dz_img;
  const uint16_t* dlt_img;
  float* partial;  // [nsplit][P]
  int64_t P;
  const int32_t* stopped;
};

__global__ void __launch_bounds__(128, 1) k_lw_wg(const LwWgArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  if (*a.stopped) return;
  const int item = blockIdx.x;
  if (item >= a.nblocks * a.nsplit) return;
  const LwBlock bk = a.blocks[item % a.nblocks];
  const int split = item / a.nblocks;
  const int t = threadIdx.x;
  const int warp = t >> 5;
  uint8_t* s_a[2] = {smem, smem + kLwWgStage};
  uint8_t* s_b[2] = {smem + 32768, smem + kLwWgStage + 32768};
  uint8_t* s_ones = smem + 2 * kLwWgStage;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 2 * kLwWgStage + 4096);  // full[2], empty[2], final
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 6);
  if (t == 0) {
    for (int i = 0; i < 5; ++i) mbar_init(&bars[i], 1);
    fence_barrier_init();
  }
  for (int i = t; i < 16 * 128; i += 128) reinterpret_cast<__half*>(s_ones)[i] = __float2half(1.0f);
  if (warp == 0) tmem_alloc(tmem_slot, 512);
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int64_t ntiles = (a.batch + kTileM - 1) / kTileM;
  const int64_t mine = a.tile_end - a.tile_begin;
  const int64_t ts = a.tile_begin + mine * split / a.nsplit, te = a.tile_begin + mine * (split + 1) / a.nsplit;
  const bool head = bk.layer == a.depth;
  const int W = a.W;
  // sources: A = input block (features for layer 0, else activations of the layer below), B = dz (or dL/dout)
  const size_t tbytes = (size_t)kTileM * W * 2;
  const uint32_t a_bytes = (uint32_t)bk.a_rows * kTileM * 2;
  const uint32_t b_bytes = head ? (uint32_t)(kTileM * 16 * 2) : (uint32_t)tbytes;
  auto a_src = [&](int64_t tau) -> const uint8_t* {
    if (bk.layer == 0)
      return reinterpret_cast<const uint8_t*>(a.feat_img) + (size_t)tau * kTileM * a.k0 * 2 + (size_t)bk.mblk * 32768;
    return reinterpret_cast<const uint8_t*>(a.act_img) + ((size_t)(bk.layer - 1) * ntiles + tau) * tbytes +
           (size_t)bk.mblk * 32768;
  };
  auto b_src = [&](int64_t tau) -> const uint8_t* {
    if (head) return reinterpret_cast<const uint8_t*>(a.dlt_img) + (size_t)tau * kTileM * 16 * 2;
    return reinterpret_cast<const uint8_t*>(a.dz_img) + ((size_t)bk.layer * ntiles + tau) * tbytes;
  };
  if (t == 0 && te > ts) {
    const uint32_t dcol = tmem, bcol = tmem + (uint32_t)bk.n;
    const uint32_t idesc = idesc_f16(kTileM, bk.n, 1, 1);
    const uint32_t idesc_b = idesc_f16(kTileM, 16, 1, 0);   // A = dz block MN-major, B = ones K-major
    const uint32_t idesc_hb = idesc_f16(kTileM, 16, 0, 1);  // A = ones (K-major, SBO 0), B = dL/dout MN-major
    auto load = [&](int64_t tau, int st) {
      mbar_arrive_expect_tx(&bars[st], a_bytes + b_bytes);
      bulk_g2s(s_a[st], a_src(tau), a_bytes, &bars[st]);
      bulk_g2s(s_b[st], b_src(tau), b_bytes, &bars[st]);
    };
    load(ts, 0);
    if (ts + 1 < te) load(ts + 1, 1);
    uint32_t nfull[2] = {0, 0};
    for (int64_t tau = ts; tau < te; ++tau) {
      const int st = (int)((tau - ts) & 1);
      mbar_wait(&bars[st], nfull[st] & 1u);
      nfull[st]++;
      tc_fence_after();
      const uint32_t sa = smem_addr(s_a[st]), sb = smem_addr(s_b[st]);
      const bool first = tau == ts;
      // the tile's K = 16 steps as groups from single asm blocks (umma_f16_run)
      const uint32_t acc0 = first ? 0u : 1u;
      umma_f16_run(dcol, smem_desc(sa, 128, 2048), smem_desc(sb, 128, 2048), idesc, acc0, kTileM / 16, 16, 16);
      if (bk.bias_blk >= 0) {
        if (!head)
          umma_f16_run(bcol, smem_desc(sb + (uint32_t)bk.bias_blk * 32768, 128, 2048),
                       smem_desc(smem_addr(s_ones), 256, 128), idesc_b, acc0, kTileM / 16, 16, 32);
        else
          umma_f16_run(bcol, smem_desc(smem_addr(s_ones), 128, 0), smem_desc(sb, 128, 2048), idesc_hb, acc0,
                       kTileM / 16, 0, 16);
      }
      umma_commit(&bars[2 + st]);
      if (tau + 2 < te) {  // refill this stage once its MMAs are done
        mbar_wait(&bars[2 + st], (nfull[st] - 1) & 1u);
        load(tau + 2, st);
      }
    }
    umma_commit(&bars[4]);
  }
  if (te > ts) mbar_wait(&bars[4], 0);
  tc_fence_after();
  // ---- flush: lane m = input index (bias: output index)
  float* part = a.partial + (size_t)split * a.P;
  const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
  const int m = warp * 32 + (t & 31);
  const int in_idx = bk.mblk * 128 + m;
  const bool none = te <= ts;
  for (int c = 0; c < bk.n / 16; ++c) {
    float v[16];
    tmem_ld16(tmem + lane_off + c * 16, v);
    tmem_ld_wait();
    if (in_idx < bk.in_real) {
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int o = c * 16 + i;
        if (o < bk.out_real) __stcs(part + bk.w_off + (int64_t)o * bk.in_real + in_idx, none ? 0.f : v[i]);
      }
    }
  }
  if (bk.bias_blk >= 0) {
    float v[16];
    tmem_ld16(tmem + lane_off + bk.n, v);
    tmem_ld_wait();
    if (!head) {
      const int o = bk.bias_blk * 128 + m;
      if (o < bk.out_real) part[bk.b_off + o] = none ? 0.f : v[0];
    } else if (m == 0) {
      for (int k = 0; k < bk.out_real; ++k) part[bk.b_off + k] = none ? 0.f : v[k];
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 512);
}
