"""Per-stage decode timing on C2 (diagnostic)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import accept_config, make_grid, train_container  # noqa: E402
from paper_2208_04448_b200 import _lib  # noqa: E402
from paper_2208_04448_b200.decoder import DeviceModel  # noqa: E402

dev = torch.device("cuda:0")
g = make_grid("c2")
c = train_container(g, accept_config(), dev, [])
m = DeviceModel(c, dev)
for _ in range(3):
    d = m.decode(True)
torch.cuda.synchronize()
m.timer = []
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
d = m.decode(True)
e1.record()
torch.cuda.synchronize()
print("decode total ms", e0.elapsed_time(e1))
for tag, n, a, b in m.timer:
    n = int(n.item()) if hasattr(n, 'item') else int(n)
    print(" stage", tag, n, "ms", a.elapsed_time(b))
m.timer = None
lo = d.leaf_origins
n = lo.shape[0] * 512
act = torch.empty(n, dtype=torch.uint8, device=dev)
for i in range(5):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    a.record()
    m.evaluate("l0", _lib.SRC_LEAF_VOX, lo, n, _lib.OUT_L0ACTIVE, u8=act)
    b.record()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    print(f" l0 alone: gpu {a.elapsed_time(b):.3f} ms, host launch {1e3 * (t1 - t0):.3f} ms")
# voxel stage alone: the active voxels of the level-0 result (no patches applied)
act_ids, acnt = m.select(act, 1, sync=False)
vals = torch.empty(n, dtype=torch.float32, device=dev)
for i in range(5):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    m.evaluate("voxel", _lib.SRC_LEAF_VOX, lo, n, _lib.OUT_VALUE, gather=act_ids, f32=vals,
               value_scale=m.value_scale, clip=m.meta.grid_class == "sdf", count=acnt)
    b.record()
    torch.cuda.synchronize()
    print(f" voxel alone: gpu {a.elapsed_time(b):.3f} ms ({int(acnt.item())} points)")
