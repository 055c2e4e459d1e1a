"""CTA-0 timeline of mlp_eval_kernel on a streamed-weight (Table-3) net,
lattice source (diagnostic; needs `make -C csrc trace`).

    NVDB_LIB=libnvdb_b200_trace.so python tools/trace_wide.py [W m depth]

Events per engine (warp 4g): 1 = layer 0 issued, 2+l = layer l's MMAs done
(epilogue start), 20+l = epilogue of layer l done (the engine's barrier),
30+l = layer l+1's MMAs issued, 9 = tile done."""
import ctypes as C
import os
import sys
from collections import defaultdict

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("NVDB_LIB", "libnvdb_b200_trace.so")
from paper_2208_04448_b200 import _lib  # noqa: E402
from paper_2208_04448_b200.decoder import NetEvaluator  # noqa: E402
from paper_2208_04448_b200.encoder import init_mlp  # noqa: E402
from paper_2208_04448_b200.model import Activation, FourierFeatures, NetRecord  # noqa: E402

W, m, depth = (int(v) for v in sys.argv[1:4]) if len(sys.argv) > 3 else (256, 256, 3)
dev = torch.device("cuda:0")


class _E:
    def __init__(self, rec):
        self.id, self.cell, self.norm_origin, self.norm_scale = 0, (0, 0, 0), np.zeros(3), 512.0
        self.rec = rec

    def nets(self):
        return [("l1", None), ("tile", None), ("l0", self.rec), ("voxel", None)]


ff = FourierFeatures(m, 5.0, 3)
p = init_mlp(2 * m, [W] * depth, 1, Activation("sine", 3.0), "binary", 4)
ev = NetEvaluator([_E(NetRecord(p, ff))], 512, 8, 0.0, dev)
nl = 16384
lo = (torch.randint(0, 64, (nl, 3), device=dev, dtype=torch.int32) * 8).contiguous()
u8 = torch.empty(nl * 512, dtype=torch.uint8, device=dev)
run = lambda: ev.evaluate("l0", _lib.SRC_LEAF_VOX, lo, nl * 512, _lib.OUT_L0ACTIVE, u8=u8)  # noqa: E731
run()
torch.cuda.synchronize()
cap = 1 << 14
buf = torch.zeros(2 * cap * 24, dtype=torch.int64, device=dev)
L = _lib.lib()
L.nvdb_debug_trace.argtypes = [C.c_void_p, C.c_uint32]
assert L.nvdb_debug_trace(C.c_void_p(buf.data_ptr()), cap) == 0
run()
torch.cuda.synchronize()
L.nvdb_debug_trace(None, 0)
a = buf.cpu().numpy().reshape(-1, 2)
a = a[a[:, 0] != 0]
a = a[np.argsort(a[:, 0], kind="stable")]
clk = a[:, 0] - a[0, 0]
evs = (a[:, 1] >> 32).astype(int)
tile = ((a[:, 1] >> 8) & 0xFFFFFF).astype(int)
warp = (a[:, 1] & 0xFF).astype(int)
rows = defaultdict(dict)
for c_, e_, t_, w_ in zip(clk, evs, tile, warp):
    rows[(w_ // 4, t_)][e_] = c_
print(f"W={W} m={m} depth={depth}: CTA0 span {clk[-1]} clk, {len([k for k in rows if 9 in rows[k]])} tiles")
print("eng  tile | start->L0 issued ->L0 done ->epi0 done ->L1 issued ->L1 done ->epi1 done ->L2 issued ->L2 done ->tile done")
prev = {}
for k in sorted(rows, key=lambda k: min(rows[k].values()))[:24]:
    r = rows[k]
    b = prev.get(k[0], 0)
    seq = [r.get(e) for e in (1, 2, 20, 30, 3, 21, 31, 4, 9)]
    out, last = [], b
    for s in seq:
        out.append(f"{(s - last) if s is not None else -1:9d}")
        last = s if s is not None else last
    print(f"{k[0]:3d} {k[1]:5d} | " + " ".join(out))
    prev[k[0]] = r.get(9, b)
