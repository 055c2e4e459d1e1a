"""C3-shaped decode throughput: fBm density 1024^3 generated on
the GPU, decomposed into 8 experts (2x2x2 at S = 512), Chameleon-class nets
(L1 3x128/m128, L0 and voxel 3x256/m256; sine, omega 3) with random weights
(the bench contract of the task -- not BASELINE.md -- asks for random-init
weights of the named architecture when no trained ones exist), then the device decode
stages over the grid's true topology: level-0 classification of every leaf
voxel and voxel regression of every active voxel, gate-blended across the
overlapping experts.

    python tools/bench_c3.py [size] [--shards N]
"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2208_04448_b200 import _lib  # noqa: E402
from paper_2208_04448_b200.decoder import NetEvaluator  # noqa: E402
from paper_2208_04448_b200.encoder import decompose, expert_norm, init_mlp  # noqa: E402
from paper_2208_04448_b200.model import Activation, EncodedSubdomain, FourierFeatures, NetRecord  # noqa: E402
from paper_2208_04448_b200.procgen import fbm_density  # noqa: E402

size = int(sys.argv[1]) if len(sys.argv) > 1 and not sys.argv[1].startswith("-") else 1024
dev = torch.device("cuda:0")
t0 = time.perf_counter()
g = fbm_density(octaves=5, lacunarity=2.0, gain=0.5, base_frequency=4.0 / 1024.0, seed=9,
                domain=((0, 0, 0), (size, size, size)), threshold=0.45)
tgen = time.perf_counter() - t0
layout = decompose(g, 512)
rng = np.random.default_rng(0)


def net(m, width, out, head, seed):
    p = init_mlp(2 * m, [width] * 3, out, Activation("sine", 3.0), head, seed)
    w, b = p.layers[-1]
    p.layers[-1] = (rng.normal(0, 0.2, size=w.shape).astype(np.float32), b)
    return NetRecord(p, FourierFeatures(m, 10.0, seed + 1))


experts = []
for sub in layout.subdomains:
    no, ns = expert_norm(sub, g)
    e = EncodedSubdomain(sub.id, sub.cell, sub.cluster_id, no, ns, 1.0)
    e.l1_classifier = net(128, 128, 3, "logits", 10 * sub.id + 1)
    e.l0_classifier = net(256, 256, 1, "binary", 10 * sub.id + 2)
    e.voxel_regressor = net(256, 256, 1, "linear", 10 * sub.id + 3)
    experts.append(e)
ev = NetEvaluator(sorted(experts, key=lambda e: e.id), layout.size, layout.halo, 0.0, dev)
lo = torch.from_numpy(g.leaf_origins.astype(np.int32)).to(dev)
nl = lo.shape[0]
nvox = nl * 512
act_ids = torch.from_numpy(np.flatnonzero(g.leaf_active.reshape(-1)).astype(np.int64)).to(dev)
na = act_ids.numel()
u8 = torch.empty(nvox, dtype=torch.uint8, device=dev)
vals = torch.empty(na, dtype=torch.float32, device=dev)


def l0():
    ev.evaluate("l0", _lib.SRC_LEAF_VOX, lo, nvox, _lib.OUT_L0ACTIVE, u8=u8)


def vox():
    ev.evaluate("voxel", _lib.SRC_LEAF_VOX, lo, na, _lib.OUT_VALUE, gather=act_ids, f32=vals)


def timed(fn):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


ms0, ms1 = timed(l0), timed(vox)
F = 2 * (512 * 256 + 2 * 256 * 256 + 256)
print(json.dumps({"workload": f"C3-shaped fBm {size}^3, 8 experts, Chameleon nets (random weights)",
                  "generate_s": round(tgen, 2), "leaves": nl, "leaf_voxels": nvox, "active_voxels": na,
                  "l0_ms": round(ms0, 2), "voxel_ms": round(ms1, 2),
                  "decode_voxels_per_s": nvox / ((ms0 + ms1) * 1e-3),
                  "tflops_per_expert_eval": round(F * (nvox + na) / ((ms0 + ms1) * 1e-3) / 1e12, 1)}))
