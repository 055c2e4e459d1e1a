"""C5-shaped random access (BASELINE configs[4]): 1e9 uniform
int32 coordinates in [0, 2048)^3 (torch Philox, seed 0) through the hybrid
grid of a 2048^3 narrow-band sphere (radius 960, half width 3: 69.5 M active
voxels): upper-tree lookup, gate-blended voxel regressor (Lucy-class 3x256 /
m256 nets with random weights: the bench contract of the task -- not
BASELINE.md -- asks for random-init weights of the named architecture), value
finalize.  The topology is the grid's own (what a perfectly trained
classifier pair would reconstruct); the query cost does not depend on the
weight values, since the explicit topology alone decides which rows reach
the regressor (decoder.py:243).

Reports the lookup's HBM roofline (18 B per query) and the regressor's
tensor rate, and times the stock svcodec ``HybridGrid.query`` (baseline/_ref)
on the first 10^6 coordinates of the same stream on the host cores.

    python tools/bench_c5.py [n_queries]
"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2208_04448_b200.decoder import NetEvaluator, hybrid_query  # noqa: E402
from paper_2208_04448_b200.encoder import decompose, expert_norm, init_mlp  # noqa: E402
from paper_2208_04448_b200.model import EncodedSubdomain, FourierFeatures, NetRecord, Activation  # noqa: E402
from paper_2208_04448_b200.procgen import sphere_sdf  # noqa: E402
from paper_2208_04448_b200.tree import DeviceTree  # noqa: E402

nq = int(float(sys.argv[1])) if len(sys.argv) > 1 else 1_000_000_000
dev = torch.device("cuda:0")
t0 = time.perf_counter()
g = sphere_sdf((1024.0, 1024.0, 1024.0), 960.0, 1.0, 3.0)
tgen = time.perf_counter() - t0
layout = decompose(g, 512)
rng = np.random.default_rng(0)
experts = []
for sub in layout.subdomains:
    no, ns = expert_norm(sub, g)
    e = EncodedSubdomain(sub.id, sub.cell, sub.cluster_id, no, ns, 3.0)
    p = init_mlp(512, [256] * 3, 1, Activation("sine", 3.0), "linear", 100 + sub.id)
    w, b = p.layers[-1]
    p.layers[-1] = (rng.normal(0, 0.2, size=w.shape).astype(np.float32), b)
    e.voxel_regressor = NetRecord(p, FourierFeatures(256, 10.0, 200 + sub.id))
    experts.append(e)
ev = NetEvaluator(sorted(experts, key=lambda e: e.id), layout.size, layout.halo, float(g.background), dev)
tree = DeviceTree(g)
gen = torch.Generator(device=dev)
gen.manual_seed(0)
coords = torch.randint(0, 2048, (nq, 3), dtype=torch.int32, device=dev, generator=gen)


def run():
    return hybrid_query(tree, ev, coords, 3.0, True)


_, _, nr = run()
torch.cuda.synchronize()


def timed(fn, reps=5):
    """median of reps device-timed calls (after the warm call above)"""
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


ms = timed(run)
ms_lookup = timed(lambda: tree.lookup(coords))
peaks = {"hbm_gbs": 6549.4, "bf16_tflops": 1641.1}
try:
    with open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")) as f:
        peaks.update(json.load(f))
except Exception:  # noqa: BLE001
    pass
F = 2 * (512 * 256 + 2 * 256 * 256 + 256)
lookup_gbs = nq * 18 / (ms_lookup * 1e-3) / 1e9
# the regressor share of the query: time beyond the lookup, flops of the rows it evaluated
reg_tflops = int(nr) * F / max((ms - ms_lookup) * 1e-3, 1e-9) / 1e12
cpu = None
if "--no-cpu" not in sys.argv:
    try:
        ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        for pth in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
            if os.path.isdir(os.path.join(pth, "svcodec")):
                sys.path.append(pth)
                break
        from svcodec.config import TrainConfig
        from svcodec.container import deserialize_container, serialize_container
        from svcodec.decoder import HybridGrid as RefHybrid
        from paper_2208_04448_b200.encoder import build_upper_tree
        from paper_2208_04448_b200.model import GridMeta, NeuralGridContainer, PatchList
        for e in experts:
            e.patches = PatchList()
        ours = NeuralGridContainer(GridMeta(g.grid_class, g.background, g.voxel_size, g.half_width, 3.0),
                                   build_upper_tree(g), layout, experts,
                                   TrainConfig(subdomain_size=512, l1_net=(3, 128), tile_net=None, l0_net=(3, 256),
                                               voxel_net=(3, 256), activation="sine", frequency=3.0,
                                               ffm_scale=10.0, ffm_size=256), 32)
        ref_c = deserialize_container(serialize_container(ours))
        topo = g.to_svcodec()
        h = RefHybrid(container=ref_c, topology=topo)
        q = coords[:1_000_000].cpu().numpy().astype(np.int64)
        t1 = time.perf_counter()
        v, a = h.query(q)
        dt = time.perf_counter() - t1
        cpu = {"value": q.shape[0] / dt, "unit": "queries/s", "cores": os.cpu_count(), "kind": "reference",
               "sample": f"svcodec HybridGrid.query (stock, baseline/_ref) on the first 10^6 coords of the same "
                         f"stream ({h.regressor_evaluations} regressor rows), {dt:.1f} s"}
    except Exception as ex:  # noqa: BLE001
        cpu = {"error": repr(ex)[:300]}
print(json.dumps({"workload": "C5-shaped: 2048^3 sphere (r 960, band 3), Lucy-class voxel nets (random weights), "
                              f"{len(experts)} experts", "generate_s": round(tgen, 1),
                  "active_voxels": int(g.leaf_active.sum()), "leaves": int(g.leaf_origins.shape[0]),
                  "queries": nq, "regressor_rows": int(nr), "ms": round(ms, 2),
                  "queries_per_s": nq / (ms * 1e-3), "lookup_ms": round(ms_lookup, 2),
                  "lookup_queries_per_s": nq / (ms_lookup * 1e-3),
                  "roofline": {"bound": "hbm", "kernel": "k_lookup", "bytes_per_query": 18,
                               "achieved": lookup_gbs, "peak": float(peaks["hbm_gbs"]), "unit": "GB/s",
                               "frac": lookup_gbs / float(peaks["hbm_gbs"])},
                  "regressor": {"bound": "tensor", "rows": int(nr), "flops_per_row": F, "achieved": reg_tflops,
                                "peak": float(peaks["bf16_tflops"]), "unit": "TFLOP/s",
                                "frac": reg_tflops / float(peaks["bf16_tflops"]),
                                "note": "query time beyond the lookup; includes select/finalize"},
                  "cpu_baseline": cpu}))
