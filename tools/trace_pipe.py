"""Absolute timeline of pipeline 0 (producer leader warp 0, epilogue leader warp 4)."""
import sys
import numpy as np
a = np.load(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/trace_l0.npy")
clk = a[:, 0] - a[0, 0]
ev = (a[:, 1] >> 32).astype(int)
tile = ((a[:, 1] >> 8) & 0xFFFFFF).astype(int)
warp = (a[:, 1] & 0xFF).astype(int)
names = {80: "I wait-full", 81: "I full-ok", 82: "I issued", 83: "I wait-rfree", 84: "I rfree-ok", 72: "P arrived-full",70: "P slot-wait", 71: "P slot-ok", 72: "P chunk-built", 73: "P bar-done", 74: "P mma-issued",
         1: "P tile-L0-issued", 2: "E l0-ready", 3: "E l1-ready", 4: "E l2-ready", 9: "E tile-done"}
sel = np.isin(warp, [0, 4, 16])
c, e, t = clk[sel], ev[sel], tile[sel]
o = np.argsort(c, kind="stable")
c, e, t = c[o], e[o], t[o]
start = np.searchsorted(c, c[len(c) // 3])
prev = c[start]
for i in range(start, min(len(c), start + 200)):
    print(f"{c[i]:9d} (+{c[i] - prev:5d}) tile {t[i]:6d} {names.get(e[i], e[i])}")
    prev = c[i]
