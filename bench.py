#!/usr/bin/env python
"""Benchmark of the NeuralVDB hot path on B200 (one JSON line on rank 0).

BASELINE.json metric: "decoded voxels/s and train samples/s at 1/2/4/8 B200;
% tensor-core peak".  Default workload = configs[1] (C2): synthetic torus
narrow-band SDF at 512^3 (gen_torus_sdf(160, 64, 1, 3) centred at 256^3,
2,424,980 active voxels, 12,983 leaves), full training of the level-1,
level-0 and voxel networks with ACCEPT_CONFIG (test_acceptance.py:72-78) on
the GPU, then whole-volume decode.

* a "step" = one whole-volume decode of the trained container (device
  resident, L2 flushed between steps); ``value`` = decoded leaf voxels/s;
* ``train`` = samples/s over the complete device-resident training of the
  three networks (800 epochs, early stops included), timed once;
* ``e2e`` = the same decode metric through the public API
  ``decode_full(container)`` from host objects to a host grid.

    python bench.py --gpus N --steps K --warmup W [--impl reference] [--workload c2|c1]

N>1 (torchrun, or spawned by bench.py itself when WORLD_SIZE is unset):
ONE workload is sharded over the ranks (strong scaling):
every net trains data parallel (1/N of each epoch's batch per rank, one
packed gradient+loss NCCL all-reduce per epoch, graph-replayed), the decode
splits the leaves into N contiguous ranges after a redundant level-1 pass
(no collective; e2e gathers the blocks on rank 0), queries split the
coordinate stream into N slices.  Times are the max over ranks.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}
TORUS = dict(major=160.0, minor=64.0, voxel=1.0, half_width=3.0, center=(256.0, 256.0, 256.0))


def load_traffic():
    """dram__bytes_read.sum + dram__bytes_write.sum of one L0-stage mlp_eval_kernel
    launch from the committed ncu --set full capture (profiles/), or None."""
    path = os.path.join(ROOT, "profiles", "r02", "ncu_mlp_eval_c2_l0_r02g.json")
    try:
        with open(path) as f:
            rec = json.load(f)[0]
        unit = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        tot = 0.0
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            v, u = rec[k].split()
            tot += float(v) * unit[u]
        return {"bytes_per_launch": tot, "launch": "L0 classifier stage, C2 (6,647,296 points)",
                "source": os.path.relpath(path, ROOT)}
    except Exception:  # noqa: BLE001
        return None


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:  # noqa: BLE001
        return PEAKS_FALLBACK, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.lines, self.proc = index, [], None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except Exception:  # noqa: BLE001
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is not None:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:  # noqa: BLE001
                self.proc.kill()
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def fwd_flops(net) -> int:
    """2*sum(in*out) incl. the head."""
    return int(sum(2 * w.shape[0] * w.shape[1] for w, _ in net.params.layers))


def transcendentals(net) -> int:
    """MUFU co-bound per point of a forward pass: 2m Fourier
    features + depth*width activations (sine nets; relu/tanh nets count 2m)."""
    hidden = net.params.layers[:-1]
    acts = sum(w.shape[0] for w, _ in hidden) if net.params.activation.kind == "sine" else 0
    return int(2 * net.ff.m + acts)


MUFU_LANES_PER_CLK_SM = 16  # measured, tools/ubench/mufu.cu (sin/ex2/tanh)


def train_flops(layers) -> int:
    """2*(3*sum MAC - MAC_0): forward + wgrad + dgrad except layer 0."""
    macs = [w.shape[0] * w.shape[1] for w, _ in layers]
    return int(2 * (3 * sum(macs) - macs[0]))


def accept_config():
    from paper_2208_04448_b200.encoder import TrainConfig
    return TrainConfig(subdomain_size=512, l1_net=(3, 48), tile_net=None, l0_net=(3, 96), voxel_net=(3, 96),
                       activation="sine", frequency=3.0, ffm_scale=5.0, ffm_size=192, lr=1e-3, decay=0.975,
                       interval=100.0, max_epochs=800, sample_interval=1, batch_size=65536,
                       significance_threshold=0.0, strict_topology=False, seed=4242)


def dragon_config():
    """SURVEY.md §8(d) C2 throughput nets, the Table-3 "Dragon" row
    (PAPER.md:430-443): L1 3x64, L0/voxel 3x128, sine/1.5, ffm 10/256."""
    from paper_2208_04448_b200.encoder import TrainConfig
    return TrainConfig(subdomain_size=512, l1_net=(3, 64), tile_net=None, l0_net=(3, 128), voxel_net=(3, 128),
                       activation="sine", frequency=1.5, ffm_scale=10.0, ffm_size=256, lr=1e-3, decay=0.975,
                       interval=100.0, max_epochs=800, sample_interval=1, batch_size=65536,
                       significance_threshold=0.0, strict_topology=False, seed=4242)


def c2_dragon(grid, dev, steps, peaks):
    """C2 with the survey's throughput nets (Dragon shape):
    the same encode() path trains them on the device (layer-streamed kernels:
    3x128/m256 exceeds the fused narrow kernel), then the whole-volume decode
    is device-timed like the headline (L2 flushed between steps); the
    3x128 weights are streamed through the MLP kernel's weight ring."""
    import torch
    from paper_2208_04448_b200.decoder import DeviceModel
    timings = []
    train_container(grid, _short(dragon_config()), dev, [])  # untimed warm-up (kernels, streams, block cache)
    c = train_container(grid, dragon_config(), dev, timings)
    m = DeviceModel(c, dev)
    for _ in range(3):
        d = m.decode(True)
    torch.cuda.synchronize()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    ts = []
    for _ in range(max(steps, 3)):
        flush.random_(0, 255)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        d = m.decode(True)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = statistics.median(ts)
    nvox, nact = d.leaf_count * 512, d.regressor_evaluations
    e = c.experts[0]
    F = {t: fwd_flops(n) for t, n in e.nets() if n is not None}
    flop = m.n1 * 4096 * F["l1"] + nvox * F["l0"] + nact * F["voxel"]
    tms = sum(t["ms"] for t in timings)
    tflop = sum(t["epochs"] * t["batch"] * t["flops_per_sample"] for t in timings)
    tsamp = sum(t["epochs"] * t["batch"] for t in timings)
    m.close()
    return {"workload": "C2 torus 512^3, Dragon nets (L1 3x64/m128, L0+voxel 3x128/m256, sine 1.5, ffm 10, "
                        "800 epochs, B=65536) trained by encode(), whole-volume decode",
            "leaf_voxels": nvox, "active_voxels": nact, "decode_ms": ms, "decode_voxels_per_s": nvox / (ms * 1e-3),
            "decode_tflops": flop / (ms * 1e-3) / 1e12,
            "decode_frac": flop / (ms * 1e-3) / 1e12 / float(peaks["bf16_tflops"]),
            "train": {"samples_per_s": tsamp / (tms * 1e-3), "ms": tms, "tflops": tflop / (tms * 1e-3) / 1e12,
                      "frac_sustained": tflop / (tms * 1e-3) / 1e12 / float(peaks["bf16_tflops_sustained"]),
                      "nets": [{k: v for k, v in t.items()} for t in timings]}}


def make_grid(workload):
    from paper_2208_04448_b200.procgen import sphere_sdf, torus_sdf
    if workload == "c1":
        return sphere_sdf((63.5, 63.5, 63.5), 61.0, 1.0, 3.0)
    t = TORUS
    return torus_sdf(t["major"], t["minor"], t["voxel"], t["half_width"], center=t["center"])


def _short(cfg, epochs: int = 16):
    """The same config with a few epochs: an untimed warm-up run."""
    import dataclasses
    return dataclasses.replace(cfg, max_epochs=epochs)


def train_container(grid, cfg, dev, timings, group=None):
    """encode() with the three trainings timed on the device (l1, tile, l0, voxel).
    ``group`` (N > 1 ranks): every net trains data parallel, each rank a 1/N
    slice of every epoch's batch, one packed all-reduce per epoch."""
    import torch
    from paper_2208_04448_b200.encoder import (DeviceTrainer, build_upper_tree, decompose, extract_patches,
                                               gather_expert_data, init_mlp, net_spec, run_concurrent,
                                               stable_seed, value_scale_of, NET_TAGS)
    from paper_2208_04448_b200.model import (Activation, EncodedSubdomain, FourierFeatures, GridMeta,
                                             NetRecord, NeuralGridContainer)
    layout = decompose(grid, cfg.subdomain_size)
    experts = []
    for sub in layout.subdomains:
        scale = value_scale_of(grid)
        data = gather_expert_data(grid, sub, scale)
        ex = EncodedSubdomain(sub.id, sub.cell, sub.cluster_id, data.norm_origin, data.norm_scale, scale)
        jobs = []
        for tag, x, y, attr in (("l1", data.l1_inputs, data.l1_labels, "l1_classifier"),
                                ("tile", data.tile_inputs, data.tile_targets, "tile_regressor"),
                                ("l0", data.l0_inputs, data.l0_labels, "l0_classifier"),
                                ("voxel", data.vox_inputs, data.vox_targets, "voxel_regressor")):
            spec = net_spec(tag, cfg)
            if spec is None or x is None:
                continue
            tid = NET_TAGS[tag]
            ff = FourierFeatures(spec.m, cfg.ffm_scale, stable_seed(cfg.seed, sub.id, tid, 0))
            p0 = init_mlp(2 * spec.m, [spec.arch[1]] * spec.arch[0], spec.out_dim,
                          Activation(cfg.activation, cfg.frequency), spec.head, stable_seed(cfg.seed, sub.id, tid, 1))
            sampled = (not spec.full_batch) and x.shape[0] > cfg.batch_size
            tr = DeviceTrainer(p0, ff, x, y, spec.loss_kind, cfg, cfg.lr, stable_seed(cfg.seed, sub.id, tid, 2),
                               sampled, spec.loss_target, dev, group=group)
            batch = cfg.batch_size if sampled else x.shape[0]
            jobs.append((tag, attr, tr, ff, int(batch), train_flops(p0.layers)))
        # the expert's nets train at once, each on its own stream with its full
        # grid (encode()'s schedule, run_concurrent); timed as one group
        torch.cuda.synchronize(dev)
        if group is not None:
            import torch.distributed as dist
            dist.barrier(group)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        res = run_concurrent([j[2] for j in jobs])
        e1.record()
        e1.synchronize()
        for (tag, attr, tr, ff, batch, fl), (loss, epochs) in zip(jobs, res):
            timings.append({"tag": tag, "epochs": epochs, "batch": batch, "ms": e0.elapsed_time(e1) / len(jobs),
                            "loss": loss, "flops_per_sample": fl, "concurrent": len(jobs)})
            setattr(ex, attr, NetRecord(tr.weights(), ff, loss, epochs))
            tr.close()
        experts.append(ex)
    extract_patches(grid, layout, experts, cfg, dev)
    meta = GridMeta(grid.grid_class, grid.background, grid.voxel_size, grid.half_width, value_scale_of(grid))
    return NeuralGridContainer(meta, build_upper_tree(grid), layout, experts, cfg, 16)


def query_bench(m, dev, steps, nq=1 << 27, lo=-32, hi=544, seed=0, rank=0, world=1):
    """Random-access point queries (SURVEY.md §8(d) C5 shape, on this workload's
    grid): uniform int32 coords in [lo, hi)^3 through HybridGrid.query_device
    (lookup K1 + gate-blended voxel regressor on the rows that resolve to an
    active leaf voxel).  Also times the lookup kernel alone for its HBM
    roofline (18 B per query: 12 B coords in, f32 value + u8 active + u8 kind out)."""
    import torch
    from paper_2208_04448_b200.decoder import HybridGrid
    hg = HybridGrid(m, m.decode(False))
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    coords = torch.randint(lo, hi, (nq, 3), dtype=torch.int32, device=dev, generator=g)
    # N ranks: each queries its contiguous 1/N slice of the same stream
    from paper_2208_04448_b200.decoder import shard_range
    qlo, qhi = shard_range(nq, rank, world)
    mine = coords[qlo:qhi]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def timed(fn):
        for _ in range(2):
            fn()
        ts = []
        for _ in range(max(steps, 3)):
            flush.random_(0, 255)
            _barrier(world)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            e1.synchronize()
            ts.append(_max_over_ranks(e0.elapsed_time(e1), dev, world))
        return statistics.median(ts)

    # end to end through the public HybridGrid.query: host int32 coords in,
    # host (value, active) out, copies inside the timed region
    ne = 1 << 24
    host = coords[:ne].cpu().numpy()
    grp = _group(world)
    for _ in range(2):
        hg.query(host, group=grp)
    te = []
    for _ in range(max(steps, 3)):
        torch.cuda.synchronize()
        _barrier(world)
        t0 = time.perf_counter()
        hg.query(host, group=grp)
        torch.cuda.synchronize()
        te.append(_max_over_ranks(time.perf_counter() - t0, dev, world))
    e2e = {"value": ne / statistics.median(te), "unit": "queries/s", "queries": ne,
           "h2d_bytes_per_step": int(host.nbytes // world), "d2h_bytes_per_step": int(ne * 5),
           "api": "HybridGrid.query(numpy int32 (n, 3), group) -> numpy (value f32, active bool) on rank 0"}
    t_lookup = timed(lambda: hg.tree.lookup(mine))
    hg.regressor_evaluations = 0
    t_query = timed(lambda: hg.query_device(mine))
    evals = hg.regressor_evaluations / (2 + max(steps, 3))
    bytes_q = 18
    return {"value": nq / (t_query * 1e-3), "unit": "queries/s", "queries": nq, "ms": t_query,
            "coords": f"uniform int32 in [{lo},{hi})^3 (torch Philox, seed {seed})"
                      + (f", {world} contiguous slices" if world > 1 else ""),
            "regressor_rows": int(evals), "e2e": e2e,
            "lookup": {"ms": t_lookup, "value": nq / (t_lookup * 1e-3), "unit": "queries/s",
                       "roofline": {"bound": "hbm", "bytes_per_query": bytes_q,
                                    "achieved": nq * bytes_q / (t_lookup * 1e-3) / 1e9, "unit": "GB/s"}}}


def c3_pipeline(dev, rank, world, size=1024, epochs=2500):
    """C3 (BASELINE configs[2]) end to end (tools/c3_pipeline.py): fBm density
    1024^3 generated on the GPU, encode() with the Chameleon row (8 experts at
    S = 512, L0 / voxel 3x256/m256, L1 3x128, 2500 epochs), then the full
    decode (level-1 stage, patches, leaves, finalize), IoU against the input.
    N ranks: experts train expert-parallel, the decode splits the leaves into
    N ranges (all ranks run it in-process); N = 1: a subprocess."""
    if world > 1:
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        import c3_pipeline as c3p
        import torch.distributed as dist
        return c3p.run(size, epochs, dev, dist.group.WORLD)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "c3_pipeline.py"), str(size), str(epochs)],
                         capture_output=True, text=True, timeout=1200,
                         env=dict(os.environ, CUDA_VISIBLE_DEVICES=os.environ.get("CUDA_VISIBLE_DEVICES", "")
                                  or str(dev.index or 0)))
    line = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    if not line:
        return {"error": (out.stderr or out.stdout)[-300:]}
    return json.loads(line[-1])


def c5_query(dev, nq=1_000_000_000):
    """C5 shape (BASELINE configs[4]) on one GPU: 1e9 uniform coordinates in
    [0, 2048)^3 through the hybrid grid of the 2048^3 narrow-band sphere
    (69.5 M active voxels), Lucy-class 3x256 voxel nets with random weights
    (tools/bench_c5.py)."""
    import subprocess
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "bench_c5.py"), str(nq)], capture_output=True,
                         text=True, timeout=900,
                         env=dict(os.environ, CUDA_VISIBLE_DEVICES=os.environ.get("CUDA_VISIBLE_DEVICES", "")
                                  or str(dev.index or 0)))
    line = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    return json.loads(line[-1]) if line else {"error": (out.stderr or out.stdout)[-300:]}


def c4_sequence(dev, frames=16):
    """C4 shape (BASELINE configs[3]): 16-frame moving sphere at 512^3 encoded with
    warm starts (encode_sequence on the GPU, ACCEPT nets; tools/bench_c4.py)."""
    import subprocess
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "bench_c4.py"), str(frames)],
                         capture_output=True, text=True, timeout=900,
                         env=dict(os.environ, CUDA_VISIBLE_DEVICES=os.environ.get("CUDA_VISIBLE_DEVICES", "")
                                  or str(dev.index or 0)))
    line = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    return json.loads(line[-1]) if line else {"error": (out.stderr or out.stdout)[-300:]}


def cpu_decode_sample(c, nleaf_sample=400):
    """Oracle timing on a bounded sample: the first leaves of the decode (L0 classify
    all their voxels, regress the active ones) + all level-1 slots."""
    import oracle as O
    from paper_2208_04448_b200.model import L1_LOCAL, LEAF_LOCAL
    orig = np.asarray(sorted(tuple(o) for o in c.upper_tree.l1_origins), dtype=np.int64)
    t0 = time.perf_counter()
    cen1 = (orig[:1, None, :] + (L1_LOCAL * 8.0 + 4.0)[None]).reshape(-1, 3)
    p1, cov1 = O.blended(c.layout, c.experts, cen1, "l1")
    cls = np.where(cov1, p1.argmax(1), 2)
    slots = np.flatnonzero(cls == 0)[:nleaf_sample]
    lo = orig[0] + L1_LOCAL[slots] * 8
    cen0 = (lo[:, None, :] + (LEAF_LOCAL + 0.5)[None]).reshape(-1, 3)
    p0, cov0 = O.blended(c.layout, c.experts, cen0, "l0")
    act = cov0 & (p0[:, 0] > 0.5)
    O.blended(c.layout, c.experts, cen0[act], "voxel")
    dt = time.perf_counter() - t0
    return cen0.shape[0] / dt, cen0.shape[0], dt, int(act.sum())


def cpu_train_sample(c, cfg, steps=3):
    """Oracle fused_step timing: voxel net, batch 65536, `steps` steps."""
    import oracle as O
    e = c.experts[0]
    rec = e.voxel_regressor
    st = O.TrainState([(w.copy(), b.copy()) for w, b in rec.params.layers], cfg.activation, cfg.frequency, rec.ff)
    rng = np.random.default_rng(0)
    x = rng.uniform(0.2, 0.8, size=(cfg.batch_size, 3)).astype(np.float32)
    y = rng.uniform(-1, 1, size=cfg.batch_size).astype(np.float32)
    O.train_step(st, x, y, "mse", np.float32(1e-3))
    t0 = time.perf_counter()
    for _ in range(steps):
        O.train_step(st, x, y, "mse", np.float32(1e-3))
    dt = time.perf_counter() - t0
    return steps * cfg.batch_size / dt, dt


def _import_svcodec():
    """The stock reference package: the driver's offline install under
    baseline/_ref (or the reference tree in the build container)."""
    for p in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
        if os.path.isdir(os.path.join(p, "svcodec")) and p not in sys.path:
            sys.path.append(p)
            break
    try:
        import svcodec  # noqa: F401
        return True
    except Exception:  # noqa: BLE001
        return False


def restrict_container(c, nodes: int):
    """A copy of an svcodec container holding only its first `nodes` level-1
    nodes (sorted-origin order = the reference's decode order,
    decoder.py:71): level-2 child bits, tile records, negative fills and
    patches restricted to them.  Input preparation for a bounded sample; the
    decode that runs on it is svcodec's own, unmodified."""
    import copy
    ut = c.upper_tree
    keep = sorted(tuple(o) for o in ut.l1_origins)[:nodes]
    ks = set(keep)
    out = copy.copy(c)
    nut = copy.copy(ut)
    nut.l1_origins = list(keep)
    nut.l1_tiles = {o: t for o, t in ut.l1_tiles.items() if tuple(o) in ks}
    nut.leaf_negative_fill = {o: b for o, b in ut.leaf_negative_fill.items()
                              if tuple(v & ~127 for v in o) in ks}
    nodes2 = []
    for nd in ut.l2_nodes:
        n2 = copy.deepcopy(nd)
        bits = np.zeros_like(np.asarray(n2.child_mask.bits))
        for o in keep:
            if tuple(v & ~4095 for v in o) == tuple(nd.origin):
                bits[(((o[0] & 4095) >> 7) << 10) | (((o[1] & 4095) >> 7) << 5) | ((o[2] & 4095) >> 7)] = True
        n2.child_mask.bits[:] = bits
        nodes2.append(n2)
    nut.l2_nodes = nodes2
    out.upper_tree = nut
    exps = []
    for e in c.experts:
        e2 = copy.copy(e)
        p = copy.copy(e.patches)
        p.l1 = [(o, k) for o, k in e.patches.l1 if tuple(v & ~127 for v in o) in ks]
        p.l0 = [(o, a, v) for o, a, v in e.patches.l0 if tuple(w & ~127 for w in o) in ks]
        e2.patches = p
        exps.append(e2)
    out.experts = exps
    return out


def reference_decode_sample(workload, nodes=None):
    """Stock svcodec (baseline/_ref): read_container of the workload's
    container fixture, restricted to its first level-1 nodes, then the
    reference's own decode_full.  Returns (voxels/s, leaf voxels, s, active)."""
    from svcodec.container import read_container
    from svcodec.decoder import decode_full as ref_decode_full
    name = "c1_sphere128.nvdb" if workload == "c1" else "c2_torus512.nvdb"
    c = read_container(os.path.join(ROOT, "tests", "golden", name))
    sub = restrict_container(c, nodes or (1 if workload == "c1" else 4))
    t0 = time.perf_counter()
    g = ref_decode_full(sub)
    dt = time.perf_counter() - t0
    nvox = sum(1 for _ in g.iter_leaves()) * 512
    return nvox / dt, nvox, dt, g.active_voxel_count()


def reference_train_sample(workload, steps=3):
    """Stock svcodec.neural.fused_step (neural.py:444-524) on the container's
    voxel net, B = 65536, `steps` steps."""
    from svcodec.container import read_container
    from svcodec.neural import AdamState, FusedNet, TrainWorkspace, fused_step
    name = "c1_sphere128.nvdb" if workload == "c1" else "c2_torus512.nvdb"
    c = read_container(os.path.join(ROOT, "tests", "golden", name))
    rec = c.experts[0].voxel_regressor
    params = rec.params.copy()
    net = FusedNet(params, rec.ff, AdamState(params))
    ws = TrainWorkspace()
    rng = np.random.default_rng(0)
    x = rng.uniform(0.2, 0.8, size=(65536, 3)).astype(np.float32)
    y = rng.uniform(-1, 1, size=65536).astype(np.float32)
    fused_step(net, x, y, "mse", np.float32(1e-3), ws)
    t0 = time.perf_counter()
    for _ in range(steps):
        fused_step(net, x, y, "mse", np.float32(1e-3), ws)
    dt = time.perf_counter() - t0
    return steps * 65536 / dt, dt


def run_reference(args, rank, world):
    """Reference arm: the UNMODIFIED svcodec (baseline/_ref) decoding a bounded
    sample of the same workload's container on the host cores (all of them:
    OpenBLAS default threading); rank 0 only.  Falls back to the numpy
    oracle port when the reference package is not installed."""
    if rank != 0:
        return
    steps, warm = min(args.steps, 3), min(args.warmup, 1)
    if _import_svcodec():
        kind = "reference"
        for _ in range(warm):
            reference_decode_sample(args.workload)
        vals = []
        for _ in range(steps):
            v, nvox, dt, nact = reference_decode_sample(args.workload)
            vals.append(v)
        tv, tdt = reference_train_sample(args.workload)
        sample = (f"svcodec.decoder.decode_full (stock, baseline/_ref) of the workload's container restricted to "
                  f"its first level-1 nodes: {nvox} leaf voxels, {nact} active, per step")
        tsample = f"3 svcodec.neural.fused_step of the voxel net, B=65536 ({tdt:.1f} s)"
    else:
        kind = "port"
        cfg = accept_config()
        c = _reference_container(args.workload, cfg)
        for _ in range(warm):
            cpu_decode_sample(c)
        vals = []
        for _ in range(steps):
            v, nvox, dt, nact = cpu_decode_sample(c)
            vals.append(v)
        tv, tdt = cpu_train_sample(c, cfg)
        sample = (f"{nvox} leaf voxels of the first decoded leaves per step (L0 classify + voxel regress on "
                  f"{nact} active), numpy/OpenBLAS oracle port (svcodec not installed)")
        tsample = f"3 oracle fused_steps of the voxel net, B=65536 ({tdt:.1f} s)"
    val = statistics.median(vals)
    line = {"metric": "decoded voxels/s", "value": val, "unit": "voxels/s", "n_gpus": world, "steps": steps,
            "warmup": warm, "ms_per_step": 1e3 * nvox / val, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic", "impl": "reference",
            "config": dict(_config(args.workload), same_config=kind == "reference"),
            "cpu_baseline": {"value": val, "unit": "voxels/s", "cores": os.cpu_count(), "kind": kind,
                             "sample": sample},
            "train": {"value": tv, "unit": "samples/s", "sample": tsample},
            "e2e": {"value": val, "unit": "voxels/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _reference_container(workload, cfg):
    """The container the oracle-port fallback decodes: the committed C1
    fixture (the reference's own AC4 encode, tests/golden/c1_sphere128.npz);
    used only when svcodec itself is not installed."""
    from paper_2208_04448_b200.model import container_from_arrays
    z = np.load(os.path.join(ROOT, "tests", "golden", "c1_sphere128.npz"))
    return container_from_arrays(z)


def _config(workload):
    if workload == "c1":
        return {"workload": "C1 sphere 128^3 narrow-band SDF, ACCEPT_CONFIG train + whole-volume decode"}
    t = TORUS
    return {"workload": f"C2 torus 512^3 narrow-band SDF (R={t['major']}, r={t['minor']}, band 3), "
                        "ACCEPT_CONFIG train (l1 3x48/m96, l0+voxel 3x96/m192, 800 epochs, B=65536) "
                        "+ whole-volume decode"}


def _group(world):
    if world <= 1:
        return None
    import torch.distributed as dist
    return dist.group.WORLD


def _barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def _max_over_ranks(v: float, dev, world: int) -> float:
    if world <= 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def spawn_ranks(n: int) -> int:
    """`bench.py --gpus N` without torchrun: launch N ranks (one per GPU) with
    torch.distributed.run on 127.0.0.1 and relay rank 0's output."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.run(cmd).returncode


def mufu_cobound(ntrans: float, kms: float, per_point, clocks):
    """The MUFU (sin/cos/ex2) ceiling next to the tensor one: algorithmic
    transcendentals / s against 16 lanes/clk/SM x 148 SMs x the sampled SM clock."""
    mhz = (clocks or {}).get("sm_mhz") or (clocks or {}).get("sm_max_mhz") or 1965.0
    peak = MUFU_LANES_PER_CLK_SM * 148 * float(mhz) * 1e6 / 1e12
    ach = ntrans / (kms * 1e-3) / 1e12 if kms > 0 else 0.0
    return {"bound": "mufu", "achieved": ach, "peak": peak, "unit": "T transcendentals/s", "frac": ach / peak,
            "per_point": per_point, "note": "algorithmic count (2m + depth*width per point); the lattice "
            "feature path issues fewer MUFU ops (Chebyshev recurrence along y)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c2", choices=["c1", "c2"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-c3", action="store_true", help="skip the C3 encode + sharded decode pipeline")
    ap.add_argument("--no-c5", action="store_true", help="skip the C5-shaped 1e9 random-query measurement")
    ap.add_argument("--no-c4", action="store_true", help="skip the C4-shaped warm-start sequence measurement")
    ap.add_argument("--no-dragon", action="store_true", help="skip the C2 run with the survey's Dragon nets")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args.gpus))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    import torch
    import torch.distributed as dist
    if args.impl == "reference":
        if world > 1:
            dist.init_process_group("gloo")
        run_reference(args, rank, world)
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return
    # one rank per GPU; NVDB_BENCH_BACKEND=gloo lets N ranks share fewer GPUs
    # (a functional check of the N > 1 path on a 1-GPU box, never a bench number)
    backend = os.environ.get("NVDB_BENCH_BACKEND", "nccl")
    local = local % max(torch.cuda.device_count(), 1) if backend != "nccl" else local
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    args.warmup = max(args.warmup, 3)
    from paper_2208_04448_b200 import _lib
    from paper_2208_04448_b200.decoder import DeviceModel, decode_full

    cfg = accept_config()
    grid = make_grid(args.workload)
    sampler = ClockSampler(local)
    sampler.start()
    # ---------------- training (timed on the device, once)
    timings = []
    if world > 1:
        dist.barrier()
    # untimed warm-up: a few epochs of every net (lazy module loading of the
    # epoch kernels, the training streams, the trainer block cache)
    train_container(grid, _short(cfg), dev, [], group=_group(world))
    c = train_container(grid, cfg, dev, timings, group=_group(world))
    train_ms = sum(t["ms"] for t in timings)
    train_samples = sum(t["epochs"] * t["batch"] for t in timings)
    train_flop = sum(t["epochs"] * t["batch"] * t["flops_per_sample"] for t in timings)
    # ---------------- decode steps
    m = DeviceModel(c, dev)
    flops = {t: fwd_flops(n) for t, n in c.experts[0].nets() if n is not None}
    transc = {t: transcendentals(n) for t, n in c.experts[0].nets() if n is not None}
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2
    shard = (rank, world) if world > 1 else None  # N ranks: contiguous leaf ranges of ONE decode
    for _ in range(args.warmup):
        d = m.decode(True, shard=shard)
    torch.cuda.synchronize()
    cnts = torch.tensor([d.leaf_count * 512, d.regressor_evaluations], dtype=torch.int64, device=dev)
    if world > 1:
        dist.all_reduce(cnts)
    nvox, nact = int(cnts[0].item()), int(cnts[1].item())
    L = _lib.lib()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = L.nvdb_launch_count()
    total_ms = 0.0
    m.timer = []
    prof = os.environ.get("NVDB_PROFILE_DECODE") == "1"  # ncu --profile-from-start off: timed decodes only
    if prof:
        torch.cuda.profiler.start()
    for _ in range(args.steps):
        flush.random_(0, 255)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        d = m.decode(True, shard=shard)
        e1.record()
        e1.synchronize()
        total_ms += e0.elapsed_time(e1)
    torch.cuda.synchronize()
    if prof:
        torch.cuda.profiler.stop()
    launches = (L.nvdb_launch_count() - launches0) / args.steps
    clocks = sampler.stop()
    timer, m.timer = m.timer, None
    tt = torch.tensor([total_ms, train_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    ms = float(tt[0].item()) / args.steps
    train_ms_max = float(tt[1].item())
    value = nvox / (ms * 1e-3)  # the whole volume's leaf voxels / max-over-ranks time
    kflops, ktr, kms, per_tag = 0.0, 0.0, 0.0, {}
    for tag, npts, a, b in timer:
        npts = int(npts.item()) if hasattr(npts, 'item') else int(npts)
        dt = a.elapsed_time(b)
        kms += dt
        kflops += npts * flops[tag]
        ktr += npts * transc[tag]
        s = per_tag.setdefault(tag, [0, 0.0])
        s[0] += npts
        s[1] += dt
    peaks, src = load_peaks()
    achieved = kflops / (kms * 1e-3) / 1e12
    peak = float(peaks["bf16_tflops"])
    train_tf = train_flop / (train_ms * 1e-3) / 1e12
    # ---------------- random-access queries (C5 shape on this grid)
    query = query_bench(m, dev, args.steps, rank=rank, world=world)
    query["lookup"]["roofline"]["peak"] = float(peaks["hbm_gbs"])
    query["lookup"]["roofline"]["frac"] = query["lookup"]["roofline"]["achieved"] / float(peaks["hbm_gbs"])
    # ---------------- e2e through the public API (host container -> host grid);
    # measured before the large C3-C5 workloads, so their allocations do not
    # shape the host / caching-allocator state it sees
    e2e_t = []
    h2d = sum(w.nbytes + b.nbytes for e in c.experts for _, n in e.nets() if n is not None
              for w, b in n.params.layers)
    import gc
    gc.collect()  # untimed: start the e2e loop without the garbage the sections above left
    for i in range(3 + 10):  # 3 untimed calls (pinned host blocks, first-touch), then 10 timed
        torch.cuda.synchronize()
        _barrier(world)
        t0 = time.perf_counter()
        g = decode_full(c, dev, group=_group(world))  # N ranks: sharded, gathered on rank 0
        torch.cuda.synchronize()
        dt = _max_over_ranks(time.perf_counter() - t0, dev, world)
        if i >= 3:
            e2e_t.append(dt)
    e2e = nvox / statistics.median(e2e_t)
    c3 = None
    if not args.no_c3:
        try:
            c3 = c3_pipeline(dev, rank, world)
            if "decode_tflops" in c3:
                c3["roofline"] = {"bound": "tensor", "kernel": "mlp_eval_kernel (all decode stages)",
                                  "achieved": c3["decode_tflops"], "peak": float(peaks["bf16_tflops"]),
                                  "unit": "TFLOP/s", "frac": c3["decode_tflops"] / float(peaks["bf16_tflops"])}
        except Exception as ex:  # noqa: BLE001 -- the headline line must still print
            c3 = {"error": repr(ex)[:300]}
    dragon = None
    if rank == 0 and world == 1 and args.workload == "c2" and not args.no_dragon:
        try:
            dragon = c2_dragon(grid, dev, args.steps, peaks)
        except Exception as ex:  # noqa: BLE001 -- the headline line must still print
            dragon = {"error": repr(ex)[:300]}
    c4 = None
    if rank == 0 and world == 1 and not args.no_c4:
        try:
            c4 = c4_sequence(dev)
        except Exception as ex:  # noqa: BLE001 -- the headline line must still print
            c4 = {"error": repr(ex)[:300]}
    c5 = None
    if rank == 0 and world == 1 and not args.no_c5:
        try:
            c5 = c5_query(dev)
        except Exception as ex:  # noqa: BLE001 -- the headline line must still print
            c5 = {"error": repr(ex)[:300]}
    d2h = (nvox // 512) * (512 * 4 + 512 + 12) + m.n1 * 4096 * 6
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        if _import_svcodec():  # the stock reference on this box's host cores
            v, nv, dt, na = reference_decode_sample(args.workload)
            tv, tdt = reference_train_sample(args.workload)
            cpu = {"value": v, "unit": "voxels/s", "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"svcodec.decoder.decode_full (stock, baseline/_ref) of this workload's container "
                             f"(tests/golden, trained by this arm's encode) restricted to its first level-1 "
                             f"nodes: {nv} leaf voxels, {na} active, {dt:.1f} s",
                   "train": {"value": tv, "unit": "samples/s",
                             "sample": f"3 svcodec.neural.fused_step, voxel net, B=65536, {tdt:.1f} s"}}
        else:
            v, nv, dt, na = cpu_decode_sample(c)
            tv, tdt = cpu_train_sample(c, cfg)
            cpu = {"value": v, "unit": "voxels/s", "cores": os.cpu_count(), "kind": "port",
                   "sample": f"oracle decode of the first {nv // 512} decoded leaves ({nv} leaf voxels: L0 classify "
                             f"+ voxel regress of {na} active), numpy/OpenBLAS, {dt:.1f} s",
                   "train": {"value": tv, "unit": "samples/s",
                             "sample": f"3 oracle fused_steps, voxel net, B=65536, {tdt:.1f} s"}}
    if rank == 0:
        line = {
            "metric": "decoded voxels/s", "value": value, "unit": "voxels/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f16xf16->f32 (fp32 head/Adam, f64 blend)",
            "data": "synthetic",
            "config": dict(_config(args.workload), leaf_voxels=nvox, active_voxels=nact, l1_slots=m.n1 * 4096,
                           parallelism=("1 GPU" if world == 1 else
                                        f"{world} ranks: decode = contiguous leaf ranges of one volume, queries = "
                                        "coordinate slices, training = data parallel (1 packed NCCL all-reduce "
                                        "per epoch, graph-replayed)"),
                           l2="flushed between steps (256 MiB write)"),
            "train": {"value": train_samples / (train_ms_max * 1e-3), "unit": "samples/s",
                      "ms": train_ms_max, "samples": train_samples,
                      "nets": [{k: v for k, v in t.items()} for t in timings],
                      "roofline": {"bound": "tensor", "achieved": train_tf, "peak": float(peaks["bf16_tflops_sustained"]),
                                   "unit": "TFLOP/s", "frac": train_tf / float(peaks["bf16_tflops_sustained"])}},
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved / peak, "traffic": load_traffic(), "peak_source": src,
                         "kernel": "mlp_eval_kernel (all decode stages)", "flops_per_point": flops,
                         "kernel_ms_per_step": kms / args.steps,
                         "per_stage_ms": {k: v[1] / args.steps for k, v in per_tag.items()},
                         "co_bound": mufu_cobound(ktr, kms, transc, clocks)},
            "query": query,
            "c2_dragon": dragon,
            "c3": c3,
            "c4_sequence": c4,
            "c5_query": c5,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e, "unit": "voxels/s", "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)},
            "gpu_launches": int(round(launches)),
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    m.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
