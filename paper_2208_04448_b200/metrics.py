"""Verification metrics on the device: svcodec.metrics.iou / rmse / mcd
(metrics.py:116-230) for DenseLeafGrids (or svcodec VdbGrids), computed by
``nvdb_metric_pass`` (csrc/metrics.cu) over device trees -- the parity
checks at C3 / C5 scale, where the reference's Python
metrics (per-leaf loops, np.unique over every coordinate) do not finish.

Semantics follow the reference exactly: SDF occupancy = leaf voxels with
value <= 0 plus non-positive tile extents; FOG IoU and RMSE run over the
union of the active sets with active tiles expanded (a side inactive at a
coordinate contributes its background); mCD samples the other grid by
trilinear interpolation at zero crossings along +x/+y/+z active edges and
averages |value| symmetrically (world units).  Sums are f64, reduced per
block and then in block order on the host.
"""

from __future__ import annotations

from typing import Dict

import numpy as np
import torch

from ._lib import check, lib
from .errors import SvcodecError
from .model import L1_LOCAL, DenseLeafGrid
from .tree import DeviceTree

_L2_LOCAL = np.stack([np.arange(32768) >> 10, (np.arange(32768) >> 5) & 31, np.arange(32768) & 31], axis=1)


def _as_dense(g) -> DenseLeafGrid:
    return g if isinstance(g, DenseLeafGrid) else DenseLeafGrid.from_svcodec(g)


def _tiles(g: DenseLeafGrid, sdf: bool):
    """Tile extents entering the metrics: active tiles (active sets) and, for
    SDF grids, non-positive tiles (occupied set); metrics.py:45-89."""
    org, ext, val, act = [], [], [], []
    for k, (v, a) in g.root_tiles.items():
        if a or (sdf and v <= 0.0):
            raise SvcodecError("root-level active/occupied tiles are not supported by metrics")
    for n in range(g.l2_origins.shape[0]):
        sel = ~g.l2_child[n] & (g.l2_active[n] | ((g.l2_tiles[n] <= 0.0) if sdf else False))
        idx = np.flatnonzero(sel)
        if idx.size:
            org.append(g.l2_origins[n] + _L2_LOCAL[idx] * 128)
            ext.append(np.full(idx.size, 128, np.int32))
            val.append(g.l2_tiles[n][idx])
            act.append(g.l2_active[n][idx])
    for n in range(g.l1_origins.shape[0]):
        sel = ~g.l1_child[n] & (g.l1_active[n] | ((g.l1_tiles[n] <= 0.0) if sdf else False))
        idx = np.flatnonzero(sel)
        if idx.size:
            org.append(g.l1_origins[n] + L1_LOCAL[idx] * 8)
            ext.append(np.full(idx.size, 8, np.int32))
            val.append(g.l1_tiles[n][idx])
            act.append(g.l1_active[n][idx])
    if not org:
        return None
    ext = np.concatenate(ext)
    first = np.concatenate([[0], np.cumsum(ext.astype(np.int64) ** 3)])
    return (np.concatenate(org).astype(np.int32), ext, np.concatenate(val).astype(np.float32),
            np.concatenate(act).astype(np.uint8), first)


class _Side:
    def __init__(self, g, dev, sdf: bool):
        self.g = _as_dense(g)
        self.tree = DeviceTree(self.g)
        self.org = torch.from_numpy(np.ascontiguousarray(self.g.leaf_origins, dtype=np.int32)).to(dev)
        t = _tiles(self.g, sdf)
        self.tiles = None if t is None else [torch.from_numpy(np.ascontiguousarray(x)).to(dev) for x in t]

    def close(self):
        self.tree.close()


def _pass(a: _Side, b: _Side, sdf: bool, want_mcd: bool, dev) -> np.ndarray:
    nb = int(lib().nvdb_metric_partials())
    part = torch.zeros(nb, dtype=torch.float64, device=dev)
    t = a.tiles
    ptr = (lambda x: x.data_ptr()) if t is not None else (lambda x: None)
    nt = 0 if t is None else int(t[1].numel())
    check(lib().nvdb_metric_pass(a.tree.handle, a.org.data_ptr(), b.tree.handle,
                                 ptr(t[0]) if t else None, ptr(t[1]) if t else None, ptr(t[2]) if t else None,
                                 ptr(t[3]) if t else None, ptr(t[4]) if t else None, nt, int(sdf), int(want_mcd),
                                 part.data_ptr(), torch.cuda.current_stream(dev).cuda_stream), "nvdb_metric_pass")
    p = part.view(-1, 8).cpu().numpy()
    return p.sum(axis=0)  # block order (numpy pairwise over a fixed layout): deterministic


def compare(a, b, device=None, mcd: bool = True) -> Dict[str, float]:
    """IoU, RMSE and (SDF) mCD between two grids, on the device."""
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    ga, gb = _as_dense(a), _as_dense(b)
    if ga.voxel_size != gb.voxel_size:
        raise SvcodecError(f"voxel size mismatch: {ga.voxel_size} vs {gb.voxel_size}")
    if ga.grid_class != gb.grid_class:
        raise SvcodecError(f"grid class mismatch: {ga.grid_class} vs {gb.grid_class}")
    sdf = ga.grid_class == "sdf"
    sa, sb = _Side(ga, dev, sdf), _Side(gb, dev, sdf)
    try:
        want = bool(mcd and sdf)
        pa = _pass(sa, sb, sdf, want, dev)
        pb = _pass(sb, sa, sdf, want, dev)
    finally:
        sa.close()
        sb.close()
    out: Dict[str, float] = {}
    if sdf:
        inter, union = pa[3], pa[2] + pb[2] - pa[3]
        out["iou"] = float(inter / union) if union else 1.0
    else:
        inter, union = pa[1], pa[0] + pb[0] - pa[1]
        out["iou"] = float(inter / union) if union else 1.0
    nunion = pa[0] + pb[0] - pa[1]
    out["rmse"] = float(np.sqrt((pa[4] + pa[5] + pb[5]) / nunion)) if nunion else float("nan")
    if want:
        if pa[6] == 0 or pb[6] == 0:
            raise SvcodecError("mcd requires surface samples on both grids")
        out["mcd"] = float(0.5 * pa[7] / pa[6] + 0.5 * pb[7] / pb[6])
        out["surface_points"] = (int(pa[6]), int(pb[6]))
    out["active"] = (int(pa[0]), int(pb[0]))
    return out


def iou(a, b, device=None) -> float:
    """metrics.iou (metrics.py:116-141)."""
    return compare(a, b, device, mcd=False)["iou"]


def rmse(a, b, device=None) -> float:
    """metrics.rmse (metrics.py:144-155)."""
    r = compare(a, b, device, mcd=False)["rmse"]
    if r != r:
        raise SvcodecError("rmse over an empty active-set union")
    return r


def mcd(a, b, device=None) -> float:
    """metrics.mcd (metrics.py:218-230), world units."""
    return compare(a, b, device, mcd=True)["mcd"]
