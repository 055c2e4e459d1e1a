#!/usr/bin/env python
"""Benchmark of the NeuralVDB hot path on B200 (one JSON line on rank 0).

Workload (BASELINE.json metric "decoded voxels/s and train samples/s"):
whole-volume neural decode of a synthetic narrow-band SDF level set from a
trained container; ``value`` = leaf voxels decoded per second (device-timed,
container resident in HBM, L2 flushed between steps).  The container is the
C1 configuration (sphere 128^3, ACCEPT_CONFIG, fp16 weights) trained by the
reference itself (tests/golden/c1_sphere128.npz).

    python bench.py --gpus N --steps K --warmup W [--impl reference]

N>1 runs under torchrun (one process per GPU): decode is data-parallel with
no collective (every rank decodes a full replica: weak scaling); the step
time is the max over ranks.
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


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p, "measured"
    except Exception:  # noqa: BLE001
        return PEAKS_FALLBACK, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.lines = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except Exception:  # noqa: BLE001
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is not None:
            time.sleep(0.25)
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


def mlp_flops_per_point(net) -> int:
    """Forward flops 2*sum(in*out) incl. the head."""
    return int(sum(2 * w.shape[0] * w.shape[1] for w, _ in net.params.layers))


def load_c1():
    from paper_2208_04448_b200.model import container_from_arrays
    z = np.load(os.path.join(ROOT, "tests", "golden", "c1_sphere128.npz"))
    return container_from_arrays(z)


def run_reference(args, rank):
    """CPU reference arm: the oracle restatement of svcodec.decode_full."""
    if rank != 0:
        return
    import oracle as O
    c = load_c1()
    steps, warm = min(args.steps, 3), min(args.warmup, 1)
    for _ in range(warm):
        O.decode(c)
    t = []
    nvox = 0
    for _ in range(steps):
        t0 = time.perf_counter()
        r = O.decode(c)
        t.append(time.perf_counter() - t0)
        nvox = r.leaf_origins.shape[0] * 512
    val = nvox / (sum(t) / len(t))
    cores = os.cpu_count()
    line = {"metric": "decoded voxels/s", "value": val, "unit": "voxels/s", "n_gpus": args.gpus,
            "steps": steps, "warmup": warm, "ms_per_step": 1e3 * sum(t) / len(t), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": "C1 sphere 128^3 ACCEPT_CONFIG whole-volume decode_full",
                       "leaf_voxels": nvox},
            "cpu_baseline": {"value": val, "unit": "voxels/s", "cores": cores, "kind": "port",
                             "sample": f"full C1 decode ({nvox} leaf voxels) per step, numpy/OpenBLAS"},
            "e2e": {"value": val, "unit": "voxels/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    import torch
    import torch.distributed as dist
    if world > 1:
        dist.init_process_group("nccl" if args.impl == "ours" else "gloo")
    if args.impl == "reference":
        run_reference(args, rank)
        if world > 1:
            dist.destroy_process_group()
        return
    args.warmup = max(args.warmup, 3)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    from paper_2208_04448_b200 import _lib
    from paper_2208_04448_b200.decoder import DeviceModel, decode_full

    c = load_c1()
    m = DeviceModel(c, dev)
    flops = {t: mlp_flops_per_point(n) for t, n in c.experts[0].nets() if n is not None}
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2
    for _ in range(args.warmup):
        d = m.decode(True)
    torch.cuda.synchronize()
    nvox = d.leaf_count * 512
    nact = d.regressor_evaluations
    n1 = m.n1
    sampler = ClockSampler(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    sampler.start()
    L = _lib.lib()
    launches0 = L.nvdb_launch_count()
    total_ms = 0.0
    m.timer = []
    for _ in range(args.steps):
        flush.random_(0, 255)  # evict L2 between steps (not timed)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        d = m.decode(True)
        e1.record()
        e1.synchronize()
        total_ms += e0.elapsed_time(e1)
    torch.cuda.synchronize()
    launches = (L.nvdb_launch_count() - launches0) // args.steps
    clocks = sampler.stop()
    timer, m.timer = m.timer, None
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item()) / args.steps
    value = world * nvox / (ms * 1e-3)
    # roofline of the fused MLP kernel: algorithmic flops / its own event time
    kflops, kms = 0.0, 0.0
    per_tag = {}
    for tag, npts, a, b in timer:
        dt = a.elapsed_time(b)
        kms += dt
        kflops += npts * flops[tag]
        s = per_tag.setdefault(tag, [0, 0.0])
        s[0] += npts
        s[1] += dt
    peaks, src = load_peaks()
    achieved = kflops / (kms * 1e-3) / 1e12
    peak = float(peaks["bf16_tflops"])
    # e2e: public API from the host container to a host grid, H2D/D2H included
    e2e_t = []
    h2d = sum(w.nbytes + b.nbytes for e in c.experts for _, n in e.nets() if n is not None
              for w, b in n.params.layers)
    for _ in range(max(2, min(args.steps, 5))):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        g = decode_full(c, dev)
        torch.cuda.synchronize()
        e2e_t.append(time.perf_counter() - t0)
    e2e = nvox / statistics.median(e2e_t)
    d2h = g.leaf_count * (512 * 4 + 512 + 12) + n1 * 4096 * 6
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        import oracle as O
        t0 = time.perf_counter()
        r = O.decode(c)
        dt = time.perf_counter() - t0
        cpu = {"value": r.leaf_origins.shape[0] * 512 / dt, "unit": "voxels/s", "cores": os.cpu_count(),
               "kind": "port", "sample": f"one full C1 decode ({r.leaf_origins.shape[0] * 512} leaf voxels), "
                                         f"numpy/OpenBLAS oracle, {dt:.1f} s"}
    if rank == 0:
        line = {
            "metric": "decoded voxels/s", "value": value, "unit": "voxels/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f16xf16->f32 (fp32 head, f64 blend)",
            "data": "synthetic",
            "config": {"workload": "C1 sphere 128^3 ACCEPT_CONFIG whole-volume decode (reference-trained fp16 container)",
                       "leaf_voxels": nvox, "active_voxels": nact, "l1_slots": n1 * 4096,
                       "parallelism": f"replicas x{world}", "l2": "flushed between steps (256 MiB write)"},
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved / peak, "traffic": None, "peak_source": src,
                         "kernel": "mlp_eval_kernel (all decode stages)",
                         "flops_per_point": flops, "kernel_ms_per_step": kms / args.steps,
                         "per_stage_ms": {k: v[1] / args.steps for k, v in per_tag.items()}},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e, "unit": "voxels/s", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h)},
            "gpu_launches": int(launches),
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    m.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
