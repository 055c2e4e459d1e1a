"""Vectorized synthetic level sets written straight into DenseLeafGrid arrays.

Same construction as the reference generators (procgen.py:174-269:
``_banded_sdf_grid``, ``_fill_interior_tiles``, ``gen_sphere_sdf``,
``gen_torus_sdf``) -- f64 distances, f32 storage, band |d| < half_width*dx,
inactive signed band values, -band interior tiles at levels 2 and 1 -- but
without per-leaf Python objects, so 512^3-class inputs build in seconds.
Host-side input plumbing, not part of the hot path.
"""

from __future__ import annotations

from typing import Callable, Sequence, Tuple

import numpy as np

from .model import GRID_CLASS_SDF, L1_LOCAL, L1_SIZE, L2_SIZE, LEAF_LOCAL, LEAF_SIZE, DenseLeafGrid, local_coords

L2_LOCAL = local_coords(5)


def _canonical_leaf_order(origins: np.ndarray) -> np.ndarray:
    root = origins & ~np.int64(4095)
    a2 = (origins & 4095) >> 7
    a1 = (origins & 127) >> 3
    i2 = (a2[:, 0] << 10) | (a2[:, 1] << 5) | a2[:, 2]
    i1 = (a1[:, 0] << 8) | (a1[:, 1] << 4) | a1[:, 2]
    return np.lexsort((i1, i2, root[:, 2], root[:, 1], root[:, 0]))


def _nodes_from_leaves(lo_: np.ndarray, bg):
    """Level-1 / level-2 node arrays over canonically ordered leaf origins
    (GridBuilder.finalize order: first appearance in canonical leaf order)."""
    l1_of_leaf = lo_ & ~np.int64(127)
    if lo_.shape[0]:
        u1, first, inv1 = np.unique(l1_of_leaf, axis=0, return_index=True, return_inverse=True)
        rank1 = np.empty(len(first), np.int64)
        rank1[np.argsort(first)] = np.arange(len(first))
        l1o = u1[np.argsort(first)]
        node = rank1[inv1.reshape(-1)]
    else:
        l1o = np.zeros((0, 3), np.int64)
        node = np.zeros(0, np.int64)
    n1 = l1o.shape[0]
    l1c = np.zeros((n1, L1_SIZE), bool)
    a1 = (lo_ & 127) >> 3
    i1 = (a1[:, 0] << 8) | (a1[:, 1] << 4) | a1[:, 2]
    l1c[node, i1] = True
    l1a = np.zeros((n1, L1_SIZE), bool)
    l1t = np.full((n1, L1_SIZE), bg, np.float32)
    root_of_l1 = l1o & ~np.int64(4095)
    if n1:
        u2, first2, inv2 = np.unique(root_of_l1, axis=0, return_index=True, return_inverse=True)
        rank2 = np.empty(len(first2), np.int64)
        rank2[np.argsort(first2)] = np.arange(len(first2))
        l2o = u2[np.argsort(first2)]
        n2i = rank2[inv2.reshape(-1)]
    else:
        l2o = np.zeros((0, 3), np.int64)
        n2i = np.zeros(0, np.int64)
    n2 = l2o.shape[0]
    l2c = np.zeros((n2, L2_SIZE), bool)
    a2 = (l1o & 4095) >> 7
    i2 = (a2[:, 0] << 10) | (a2[:, 1] << 5) | a2[:, 2]
    l2c[n2i, i2] = True
    l2a = np.zeros((n2, L2_SIZE), bool)
    l2t = np.full((n2, L2_SIZE), bg, np.float32)
    return l1o, l1c, l1a, l1t, l2o, l2c, l2a, l2t


def banded_sdf_grid(distance: Callable[[np.ndarray], np.ndarray], lo_idx, hi_idx, voxel_size: float,
                    half_width: float, chunk: int = 4096, lipschitz: bool = True) -> DenseLeafGrid:
    """procgen.py:174-197 + 200-232 as array code.

    With ``lipschitz`` (true for exact SDFs such as the sphere and torus) a
    leaf block is skipped when its centre lies farther than the band plus the
    block's half-diagonal from the surface: none of its voxels can be active,
    so the reference would drop it too and the output is unchanged.
    """
    band = half_width * voxel_size
    lo = np.asarray(lo_idx, dtype=np.int64) & ~np.int64(7)
    hi = np.asarray(hi_idx, dtype=np.int64)
    axes = [np.arange(lo[a], hi[a] + 1, 8, dtype=np.int64) for a in range(3)]
    if lipschitz:
        reach = band + (3.5 * np.sqrt(3.0) + 0.01) * voxel_size
        keep = []
        for x in axes[0]:
            gy, gz = np.meshgrid(axes[1], axes[2], indexing="ij")
            slab = np.stack([np.full(gy.size, x, np.int64), gy.ravel(), gz.ravel()], axis=1)
            dc = distance((slab.astype(np.float64) + 3.5) * voxel_size)
            keep.append(slab[np.abs(dc) < reach])
        blocks = np.concatenate(keep) if keep else np.zeros((0, 3), np.int64)
    else:
        gx, gy, gz = np.meshgrid(*axes, indexing="ij")
        blocks = np.stack([gx.ravel(), gy.ravel(), gz.ravel()], axis=1)
    keep_o, keep_a, keep_v = [], [], []
    for s in range(0, len(blocks), chunk):
        blk = blocks[s:s + chunk]
        coords = (blk[:, None, :] + LEAF_LOCAL[None]).astype(np.float64)
        d = distance(coords.reshape(-1, 3) * voxel_size).reshape(len(blk), LEAF_SIZE)
        active = np.abs(d) < band
        k = active.any(axis=1)
        if not k.any():
            continue
        dk, ak = d[k], active[k]
        keep_o.append(blk[k])
        keep_a.append(ak)
        keep_v.append(np.where(ak, dk, np.where(dk < 0, -band, band)).astype(np.float32))
    if keep_o:
        lo_ = np.concatenate(keep_o)
        la = np.concatenate(keep_a)
        lv = np.concatenate(keep_v)
    else:
        lo_ = np.zeros((0, 3), np.int64)
        la = np.zeros((0, LEAF_SIZE), bool)
        lv = np.zeros((0, LEAF_SIZE), np.float32)
    order = _canonical_leaf_order(lo_)
    lo_, la, lv = lo_[order], la[order], lv[order]
    bg = np.float32(band)
    l1o, l1c, l1a, l1t, l2o, l2c, l2a, l2t = _nodes_from_leaves(lo_, bg)
    n1, n2 = l1o.shape[0], l2o.shape[0]
    # interior tiles (procgen.py:200-232): empty slots whose centre is inside
    for j in range(n2):
        empty = np.flatnonzero(~l2c[j] & ~l2a[j])
        if empty.size:
            cen = (l2o[j] + L2_LOCAL[empty] * 128).astype(np.float64) + (128 - 1) / 2.0
            d = distance(cen * voxel_size)
            l2t[j, empty[d < 0]] = -band
    for j in range(n1):
        empty = np.flatnonzero(~l1c[j] & ~l1a[j])
        if empty.size:
            cen = (l1o[j] + L1_LOCAL[empty] * 8).astype(np.float64) + (8 - 1) / 2.0
            d = distance(cen * voxel_size)
            l1t[j, empty[d < 0]] = -band
    return DenseLeafGrid(background=float(bg), grid_class=GRID_CLASS_SDF, voxel_size=float(voxel_size),
                         half_width=float(np.float32(half_width)), root_tiles={}, l2_origins=l2o, l2_child=l2c,
                         l2_active=l2a, l2_tiles=l2t, l1_origins=l1o, l1_child=l1c, l1_active=l1a, l1_tiles=l1t,
                         leaf_origins=lo_, leaf_active=la, leaf_values=lv)


def sphere_sdf(center: Sequence[float], radius: float, voxel_size: float = 1.0,
               half_width: float = 3.0) -> DenseLeafGrid:
    """gen_sphere_sdf (procgen.py:235-247)."""
    c = np.asarray(center, dtype=np.float64)

    def distance(p):
        return np.linalg.norm(p - c, axis=1) - radius

    reach = radius / voxel_size + half_width + 1
    lo = np.floor(c / voxel_size - reach).astype(np.int64)
    hi = np.ceil(c / voxel_size + reach).astype(np.int64)
    return banded_sdf_grid(distance, lo, hi, voxel_size, half_width)


def torus_sdf(major_radius: float, minor_radius: float, voxel_size: float, half_width: float,
              center: Sequence[float] = (0.0, 0.0, 0.0)) -> DenseLeafGrid:
    """gen_torus_sdf (procgen.py:250-269), z-axis torus."""
    c = np.asarray(center, dtype=np.float64)

    def distance(p):
        q = p - c
        r = np.hypot(q[:, 0], q[:, 1]) - major_radius
        return np.hypot(r, q[:, 2]) - minor_radius

    reach = (major_radius + minor_radius) / voxel_size + half_width + 1
    zreach = minor_radius / voxel_size + half_width + 1
    lo = np.floor(c / voxel_size - (reach, reach, zreach)).astype(np.int64)
    hi = np.ceil(c / voxel_size + (reach, reach, zreach)).astype(np.int64)
    return banded_sdf_grid(distance, lo, hi, voxel_size, half_width)


def fbm_density(octaves: int = 4, lacunarity: float = 2.0, gain: float = 0.5, base_frequency: float = 0.05,
                seed: int = 0, domain=((0, 0, 0), (64, 64, 64)), threshold: float = 0.5, voxel_size: float = 1.0,
                device=None) -> DenseLeafGrid:
    """gen_fbm_density (procgen.py:283-309) with the voxel work on the GPU
    (nvdb_fbm_leaves, bit-exact): every leaf block covering the domain, f64
    value-noise fBm per voxel, active = inside & value > threshold, leaves
    with an active voxel kept (values where active, else 0), FOG grid with
    background 0 and no tiles."""
    import ctypes as C

    import torch

    from . import _lib
    from .model import GRID_CLASS_FOG
    if octaves < 1:
        raise ValueError("octaves must be >= 1")
    lo = np.asarray(domain[0], dtype=np.int64)
    hi = np.asarray(domain[1], dtype=np.int64) - 1
    if (hi < lo).any():
        raise ValueError(f"empty fBm domain {domain}")
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    axes = [np.arange(lo[a] & ~np.int64(7), hi[a] + 1, 8, dtype=np.int64) for a in range(3)]
    gx, gy, gz = np.meshgrid(*axes, indexing="ij")
    blocks = np.stack([gx.ravel(), gy.ravel(), gz.ravel()], axis=1)
    nb = blocks.shape[0]
    d_blocks = torch.from_numpy(blocks.astype(np.int32)).to(dev)
    vals = torch.empty(nb * LEAF_SIZE, dtype=torch.float32, device=dev)
    act = torch.empty(nb * LEAF_SIZE, dtype=torch.uint8, device=dev)
    keep = torch.zeros(nb, dtype=torch.int32, device=dev)
    spec = _lib.FbmDesc(octaves=int(octaves), lacunarity=float(lacunarity), gain=float(gain),
                        base_frequency=float(base_frequency), seed=int(seed) & ((1 << 64) - 1),
                        lo=(C.c_int32 * 3)(*[int(v) for v in lo]), hi=(C.c_int32 * 3)(*[int(v) for v in hi]),
                        threshold=float(threshold), voxel_size=float(voxel_size))
    _lib.check(_lib.lib().nvdb_fbm_leaves(C.byref(spec), d_blocks.data_ptr(), nb, vals.data_ptr(), act.data_ptr(),
                                          keep.data_ptr(), torch.cuda.current_stream(dev).cuda_stream),
               "nvdb_fbm_leaves")
    kept = torch.nonzero(keep).squeeze(1)
    lo_ = blocks[kept.cpu().numpy()]
    la = act.view(nb, LEAF_SIZE)[kept].cpu().numpy().astype(bool)
    lv = vals.view(nb, LEAF_SIZE)[kept].cpu().numpy()
    order = _canonical_leaf_order(lo_)
    lo_, la, lv = lo_[order], la[order], lv[order]
    bg = np.float32(0.0)
    l1o, l1c, l1a, l1t, l2o, l2c, l2a, l2t = _nodes_from_leaves(lo_, bg)
    return DenseLeafGrid(background=0.0, grid_class=GRID_CLASS_FOG, voxel_size=float(voxel_size), half_width=0.0,
                         root_tiles={}, l2_origins=l2o, l2_child=l2c, l2_active=l2a, l2_tiles=l2t, l1_origins=l1o,
                         l1_child=l1c, l1_active=l1a, l1_tiles=l1t, leaf_origins=lo_, leaf_active=la,
                         leaf_values=lv)
