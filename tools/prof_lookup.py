"""k_lookup on the C2 torus tree, 2^27 uniform int32 coords in [-32, 544)^3
(the bench's query stream), for ncu (diagnostic)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import make_grid  # noqa: E402
from paper_2208_04448_b200.tree import DeviceTree  # noqa: E402

dev = torch.device("cuda:0")
t = DeviceTree(make_grid("c2"))
g = torch.Generator(device=dev)
g.manual_seed(0)
coords = torch.randint(-32, 544, (1 << 27, 3), dtype=torch.int32, device=dev, generator=g)
for _ in range(3):
    v, a, k = t.lookup(coords)
torch.cuda.synchronize()
print("kinds", torch.bincount(k.long(), minlength=3).tolist())
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
ts = []
for _ in range(15):
    flush.random_(0, 255)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    t.lookup(coords)
    e1.record()
    e1.synchronize()
    ts.append(e0.elapsed_time(e1))
ts.sort()
ms = ts[len(ts) // 2]
print(f"lookup {ms:.3f} ms = {coords.shape[0] / ms / 1e6:.1f} G q/s = {coords.shape[0] * 18 / ms / 1e6:.0f} GB/s")
