"""Per-chunk feature timeline of engine 0 (reads gpurun_out/trace_l0.npy)."""
import numpy as np
a = np.load("gpurun_out/trace_l0.npy")
clk = a[:, 0] - a[0, 0]
ev = (a[:, 1] >> 32).astype(int)
tile = ((a[:, 1] >> 8) & 0xFFFFFF).astype(int)
warp = (a[:, 1] & 0xFF).astype(int)
sel = (warp < 8) & np.isin(ev, [70, 71, 72, 73, 1, 2, 3, 4, 9])
c, e, t, w = clk[sel], ev[sel], tile[sel], warp[sel]
tiles = sorted(set(t))
T = tiles[len(tiles) // 3]
m = t == T
base = c[m].min()
last = {}
for ci, ei, wi in zip(c[m], e[m], w[m]):
    print(f"{ci - base:7d} ev {ei:3d} warp {wi}")
# per-phase totals over all tiles of engine 0
dur = {"slot wait": [], "compute": [], "barrier": []}
for T in tiles[5:-5]:
    m = t == T
    for wi in range(8):
        mm = m & (w == wi)
        ee, cc_ = e[mm], c[mm]
        s70 = cc_[ee == 70]; s71 = cc_[ee == 71]; s72 = cc_[ee == 72]; s73 = cc_[ee == 73]
        n = min(len(s70), len(s71), len(s72), len(s73))
        dur["slot wait"] += list(s71[:n] - s70[:n])
        dur["compute"] += list(s72[:n] - s71[:n])
        dur["barrier"] += list(s73[:n] - s72[:n])
for k, v in dur.items():
    print(k, "median", np.median(v), "mean", np.mean(v), "p90", np.percentile(v, 90))
