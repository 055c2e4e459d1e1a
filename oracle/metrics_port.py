"""numpy restatement of svcodec.metrics IoU and mCD -- TEST INFRASTRUCTURE ONLY.

Used to judge end-to-end quality parity (AC4: IoU >= 0.99, mCD <= 0.5 dx)
of GPU encode -> decode against the reference's recorded values.  Operates
on DenseLeafGrid via the oracle lookup.
"""

from __future__ import annotations

import numpy as np

from .svcodec_port import LEAF_OFFS, SLOT_OFFS, lookup

_L2_OFFS = np.stack([np.arange(32768) >> 10, (np.arange(32768) >> 5) & 31, np.arange(32768) & 31], axis=1)


def _expand(origin, extent):
    ax = np.arange(extent, dtype=np.int64)
    gx, gy, gz = np.meshgrid(ax, ax, ax, indexing="ij")
    return np.asarray(origin, dtype=np.int64) + np.stack([gx.ravel(), gy.ravel(), gz.ravel()], 1)


def occupied_coords(g) -> np.ndarray:
    """metrics.py:68-105: leaf voxels with value <= 0 plus non-positive tile extents."""
    parts = []
    li, vi = np.nonzero(g.leaf_values <= 0.0)
    if li.size:
        parts.append(g.leaf_origins[li] + LEAF_OFFS[vi])
    for n in range(g.l2_origins.shape[0]):
        for idx in np.flatnonzero(~g.l2_child[n] & (g.l2_tiles[n] <= 0.0)):
            parts.append(_expand(g.l2_origins[n] + _L2_OFFS[idx] * 128, 128))
    for n in range(g.l1_origins.shape[0]):
        for idx in np.flatnonzero(~g.l1_child[n] & (g.l1_tiles[n] <= 0.0)):
            parts.append(_expand(g.l1_origins[n] + SLOT_OFFS[idx] * 8, 8))
    if not parts:
        return np.zeros((0, 3), np.int64)
    return np.unique(np.concatenate(parts), axis=0)


def _packed(c):
    c = c + (1 << 20)
    return (c[:, 0] << 42) | (c[:, 1] << 21) | c[:, 2]


def iou_sdf(a, b) -> float:
    """metrics.py:116-141 (SDF branch)."""
    oa, ob = occupied_coords(a), occupied_coords(b)
    if oa.shape[0] == 0 and ob.shape[0] == 0:
        return 1.0
    pa, pb = _packed(oa), _packed(ob)
    inter = np.intersect1d(pa, pb, assume_unique=True).size
    union = pa.size + pb.size - inter
    return float(inter / union) if union else 1.0


def surface_samples(g) -> np.ndarray:
    """metrics.py:168-194: zero crossings on +x/+y/+z edges from active voxels."""
    li, vi = np.nonzero(g.leaf_active)
    coords = g.leaf_origins[li] + LEAF_OFFS[vi]
    values = g.leaf_values[li, vi]
    pts = []
    for axis in range(3):
        nb = coords.copy()
        nb[:, axis] += 1
        nv, na, _ = lookup(g, nb)
        v0, v1 = values.astype(np.float64), nv.astype(np.float64)
        cross = na & (v0 * v1 < 0.0)
        if cross.any():
            t = v0[cross] / (v0[cross] - v1[cross])
            p = coords[cross].astype(np.float64)
            p[:, axis] += t
            pts.append(p)
        zero = na & (v0 == 0.0)
        if zero.any():
            pts.append(coords[zero].astype(np.float64))
    if not pts:
        return np.zeros((0, 3))
    return np.unique(np.concatenate(pts), axis=0)


def trilinear(g, p) -> np.ndarray:
    """metrics.py:197-215."""
    base = np.floor(p).astype(np.int64)
    frac = p - base
    out = np.zeros(p.shape[0])
    for corner in range(8):
        offs = np.array([(corner >> 2) & 1, (corner >> 1) & 1, corner & 1], dtype=np.int64)
        vals, _, _ = lookup(g, base + offs)
        w = np.ones(p.shape[0])
        for ax in range(3):
            w *= frac[:, ax] if offs[ax] else 1.0 - frac[:, ax]
        out += w * vals.astype(np.float64)
    return out


def mcd(a, b) -> float:
    """metrics.py:218-230 (world units)."""
    sa, sb = surface_samples(a), surface_samples(b)
    return float(0.5 * np.abs(trilinear(b, sa)).mean() + 0.5 * np.abs(trilinear(a, sb)).mean())
