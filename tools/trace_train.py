"""CTA-0 timeline of the fused training kernel (trace build):
    NVDB_LIB=libnvdb_b200_trace.so python tools/trace_train.py [voxel|l0|l1]"""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("NVDB_LIB", "libnvdb_b200_trace.so")
from bench import accept_config, make_grid  # noqa: E402
from paper_2208_04448_b200 import _lib  # noqa: E402
from paper_2208_04448_b200.encoder import (DeviceTrainer, decompose, gather_expert_data, init_mlp,  # noqa: E402
                                           net_spec, stable_seed, value_scale_of)
from paper_2208_04448_b200.model import Activation, FourierFeatures  # noqa: E402

tag = sys.argv[1] if len(sys.argv) > 1 else "voxel"
cfg = accept_config()
g = make_grid("c2")
sub = decompose(g, 512).subdomains[0]
d = gather_expert_data(g, sub, value_scale_of(g))
x, y = {"l1": (d.l1_inputs, d.l1_labels), "l0": (d.l0_inputs, d.l0_labels),
        "voxel": (d.vox_inputs, d.vox_targets)}[tag]
spec = net_spec(tag, cfg)
ff = FourierFeatures(spec.m, cfg.ffm_scale, stable_seed(cfg.seed, 0, 3, 0))
p0 = init_mlp(2 * spec.m, [spec.arch[1]] * spec.arch[0], spec.out_dim, Activation("sine", 3.0), spec.head, 1)
tr = DeviceTrainer(p0, ff, x, y, spec.loss_kind, cfg, cfg.lr, 7, not spec.full_batch, -1.0, torch.device("cuda:0"))
tr.run(3)
torch.cuda.synchronize()
cap = 4096
buf = torch.zeros(2 * cap * 16, dtype=torch.int64, device="cuda:0")
L = _lib.lib()
L.nvdb_debug_ttrace.argtypes = [C.c_void_p, C.c_uint32]
L.nvdb_debug_ttrace(C.c_void_p(buf.data_ptr()), cap)
tr.run(1)
torch.cuda.synchronize()
L.nvdb_debug_ttrace(None, 0)
a = buf.cpu().numpy().reshape(-1, 2)
a = a[a[:, 0] != 0]
a = a[np.argsort(a[:, 0], kind="stable")]
clk = a[:, 0] - a[0, 0]
ev = (a[:, 1] >> 32).astype(int)
tile = ((a[:, 1] >> 8) & 0xFFFFFF).astype(int)
warp = (a[:, 1] & 0xFF).astype(int)
names = {1: "fb x loaded", 2: "fb L0 issued", 3: "fb L0 done", 4: "fb fwd done", 5: "fb loss done",
         6: "fb tile done", 10: "wg tile start", 11: "wg stage0 done", 12: "wg stage1", 13: "wg stage2",
         14: "wg stage3", 20: "wg mma drained", 21: "wg partials written"}
prev = 0
for c_, e_, t_, w_ in zip(clk, ev, tile, warp):
    if w_ == 0:
        print(f"{c_:8d} (+{c_ - prev:6d}) tile {t_:5d} {names.get(e_, e_)}")
        prev = c_
