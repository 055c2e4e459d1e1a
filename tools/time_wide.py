"""Throughput of the fused MLP kernel on Table-3 net shapes (random weights):
forward_block over N uniform points (per-point features) and the lattice
(leaf-voxel) source used by the L0 decode stage.

    python tools/time_wide.py [W m depth]...
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2208_04448_b200 import _lib  # noqa: E402
from paper_2208_04448_b200.encoder import init_mlp  # noqa: E402
from paper_2208_04448_b200.model import (Activation, EncodedSubdomain, FourierFeatures,  # noqa: E402
                                         NetRecord)
from paper_2208_04448_b200.netset import DeviceNetSet  # noqa: E402
from paper_2208_04448_b200.decoder import NetEvaluator  # noqa: E402

dev = torch.device("cuda:0")
shapes = [(96, 192, 3), (128, 256, 3), (192, 192, 3), (256, 256, 3)]
if len(sys.argv) > 3:
    a = [int(v) for v in sys.argv[1:]]
    shapes = [tuple(a[i:i + 3]) for i in range(0, len(a), 3)]


class _E:
    def __init__(self, rec):
        self.id, self.cell, self.norm_origin, self.norm_scale = 0, (0, 0, 0), np.zeros(3), 512.0
        self.rec = rec

    def nets(self):
        return [("l1", None), ("tile", None), ("l0", self.rec), ("voxel", None)]


def timed(fn, reps=5):
    for _ in range(2):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return min(ts)


for (W, m, depth) in shapes:
    ff = FourierFeatures(m, 5.0, 3)
    p = init_mlp(2 * m, [W] * depth, 1, Activation("sine", 3.0), "binary", 4)
    flop = 2 * sum(w.shape[0] * w.shape[1] for w, _ in p.layers)
    ns = DeviceNetSet([_E(NetRecord(p, ff))], 512)
    n = 1 << 23
    pts = torch.rand((n, 3), device=dev)
    out = torch.empty((n, 1), device=dev)
    ms = timed(lambda: ns.forward(0, pts, out))
    ns.close()
    # lattice source: leaf-voxel ids of 16384 leaves in a 512^3 box
    ev = NetEvaluator([_E(NetRecord(p, ff))], 512, 8, 0.0, dev)
    nl = 16384
    lo = (torch.randint(0, 64, (nl, 3), device=dev, dtype=torch.int32) * 8).contiguous()
    u8 = torch.empty(nl * 512, dtype=torch.uint8, device=dev)
    ms2 = timed(lambda: ev.evaluate("l0", _lib.SRC_LEAF_VOX, lo, nl * 512, _lib.OUT_L0ACTIVE, u8=u8))
    ev.close()
    print(f"W={W} m={m} depth={depth}: {flop} flop/pt; forward {n / ms / 1e6:.2f} Gpts/s "
          f"{flop * n / ms / 1e9:.0f} TFLOP/s; lattice {nl * 512 / ms2 / 1e6:.2f} Gpts/s "
          f"{flop * nl * 512 / ms2 / 1e9:.0f} TFLOP/s")
