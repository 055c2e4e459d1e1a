"""CTA-0 timeline of mlp_eval_kernel (diagnostic; needs `make -C csrc trace`).

    NVDB_LIB=libnvdb_b200_trace.so python tools/trace_eval.py [l0|voxel]

Events (clock64 of SM 0): producer 1/2/3 = ring wait begin/end, chunk
published; epilogue 10+l/20+l = layer-l wait begin/end, 30+l = layer done,
40 = tile outputs; MMA 60 = layer 0 start, 61 = chunk issued, 62 = layer 0
committed, 50+l = hidden layer l issued (tile field = group).
"""
import ctypes as C
import os
import sys
from collections import defaultdict

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("NVDB_LIB", "libnvdb_b200_trace.so")
from bench import accept_config, make_grid, train_container  # noqa: E402
from paper_2208_04448_b200 import _lib  # noqa: E402
from paper_2208_04448_b200.decoder import DeviceModel  # noqa: E402

stage = sys.argv[1] if len(sys.argv) > 1 else "l0"
dev = torch.device("cuda:0")
c = train_container(make_grid(os.environ.get("WORKLOAD", "c2")), accept_config(), dev, [])
m = DeviceModel(c, dev)
d = m.decode(True)
torch.cuda.synchronize()
lo = d.leaf_origins
n = lo.shape[0] * 512
out = torch.empty(n, dtype=torch.uint8, device=dev)
run = lambda: m.evaluate("l0", _lib.SRC_LEAF_VOX, lo, n, _lib.OUT_L0ACTIVE, u8=out)  # noqa: E731
run()
torch.cuda.synchronize()
cap = 1 << 14  # records per warp
buf = torch.zeros(2 * cap * 24, dtype=torch.int64, device=dev)
L = _lib.lib()
L.nvdb_debug_trace.argtypes = [C.c_void_p, C.c_uint32]
assert L.nvdb_debug_trace(C.c_void_p(buf.data_ptr()), cap) == 0
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
run()
e1.record()
torch.cuda.synchronize()
L.nvdb_debug_trace(None, 0)
ms = e0.elapsed_time(e1)
a = buf.cpu().numpy().reshape(-1, 2)
a = a[a[:, 0] != 0]
a = a[np.argsort(a[:, 0], kind="stable")]
t0 = a[0, 0]
clk = a[:, 0] - t0
ev = (a[:, 1] >> 32).astype(int)
tile = ((a[:, 1] >> 8) & 0xFFFFFF).astype(int)
warp = (a[:, 1] & 0xFF).astype(int)
print(f"stage {stage}: {n} points, {ms:.3f} ms, {len(a)} events, CTA0 span {clk[-1]} clk")
ntiles = len(set(tile[ev == 9]))
print(f"CTA0 tiles {ntiles}, clk per tile {clk[-1] / max(ntiles, 1):.0f}")
# per engine (warp // 4): tile phases relative to the previous tile's end
prev = {}
rows = defaultdict(list)
for c_, e_, t_, w_ in zip(clk, ev, tile, warp):
    g = w_ // 4
    rows[(g, t_)].append((e_, c_))
print("eng tile | L0 issued  l0 done  l1 done  l2 done  tile done   (clk from previous tile end)")
ends = {}
keys = sorted(rows, key=lambda k: rows[k][0][1])
for (g, t_) in keys[30:60]:
    r = dict(rows[(g, t_)])
    b = ends.get(g, min(r.values()))
    print(f"{g:3d} {t_:5d} | " + " ".join(f"{r.get(k, 0) - b:8d}" for k in (1, 2, 3, 4, 9)))
    ends[g] = r.get(9, b)
for g in range(3):
    ts = [dict(rows[k]) for k in keys if k[0] == g]
    ts = [r for r in ts if 9 in r and 1 in r]
    if len(ts) > 10:
        d = np.diff([r[9] for r in ts])
        ph = np.median([[r[1] - r.get(9, 0) for r in ts[:1]]]) if ts else 0
        print(f"engine {g}: {len(ts)} tiles, median tile period {np.median(d):.0f} clk")
np.save("gpurun_out/trace_" + stage + ".npy", a)
