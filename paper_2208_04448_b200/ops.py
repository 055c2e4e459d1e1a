"""Operator seams with the reference's signatures (numpy in, numpy out).

* ``forward_block(params, ff, pts, chunk)`` -- neural.py:527-550
* ``blended_l1_probs / blended_l0_probs / blended_values`` -- inference.py:65-84
* ``get_values(grid, coords, with_kind)`` -- grid.py:310-350

Each call uploads its inputs, runs the CUDA kernels and copies the result
back; hot loops should hold a :class:`~.decoder.DeviceModel` instead.
"""

from __future__ import annotations

from typing import Tuple

import numpy as np
import torch

from .model import DenseLeafGrid
from .netset import DeviceNetSet


def _dev() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2208_04448_b200 needs a CUDA device (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


class _OneNet:
    def __init__(self, params, ff):
        self.id, self.cell, self.norm_origin, self.norm_scale = 0, (0, 0, 0), np.zeros(3), 1.0
        from .model import NetRecord
        self._rec = NetRecord(params, ff)
        self._tag = "l1" if params.head == "logits" else "voxel"

    def nets(self):
        return [(t, self._rec if t == self._tag else None) for t in ("l1", "tile", "l0", "voxel")]


def forward_block(params, ff, pts: np.ndarray, chunk: int = 131072) -> np.ndarray:
    """Raw float32 outputs (n, out_dim) of one net at normalized points."""
    del chunk  # the kernel streams tiles itself
    pts = np.ascontiguousarray(np.asarray(pts, dtype=np.float32).reshape(-1, 3))
    if np.isnan(pts).any():
        raise ValueError("NaN in inputs")
    ns = DeviceNetSet([_OneNet(params, ff)], 512)
    try:
        out = ns.forward(0, torch.from_numpy(pts).to(_dev()))
        return out.cpu().numpy()
    finally:
        ns.close()


def _blended(layout, experts, centers, tag: str):
    centers = np.ascontiguousarray(np.asarray(centers, dtype=np.float64).reshape(-1, 3))
    ex = sorted(experts, key=lambda e: e.id)
    ns = DeviceNetSet(ex, layout.size, layout.halo)
    try:
        out, cov = ns.blended(tag, torch.from_numpy(centers).to(_dev()))
        return out.cpu().numpy(), cov.cpu().numpy().astype(bool)
    finally:
        ns.close()


def blended_l1_probs(layout, experts, centers) -> Tuple[np.ndarray, np.ndarray]:
    """(n,3) blended level-1 class probabilities + coverage (inference.py:65-68)."""
    return _blended(layout, experts, centers, "l1")


def blended_l0_probs(layout, experts, centers) -> Tuple[np.ndarray, np.ndarray]:
    """(n,) blended active probabilities + coverage (inference.py:71-75)."""
    p, c = _blended(layout, experts, centers, "l0")
    return p[:, 0], c


def blended_values(layout, experts, centers, net_name: str = "voxel") -> Tuple[np.ndarray, np.ndarray]:
    """(n,) blended regressor outputs in scaled units + coverage (inference.py:78-84)."""
    v, c = _blended(layout, experts, centers, net_name)
    return v[:, 0], c


def get_values(grid, coords, with_kind: bool = False):
    """VdbGrid.get_values (grid.py:310-350) through the device tree lookup."""
    from .tree import DeviceTree
    g = grid if isinstance(grid, DenseLeafGrid) else DenseLeafGrid.from_svcodec(grid)
    c = np.asarray(coords, dtype=np.int64).reshape(-1, 3)
    if c.size and np.abs(c).max() >= (1 << 30):
        from .errors import SvcodecError
        raise SvcodecError("coordinate outside legal range +-2^30")
    tree = DeviceTree(g)
    try:
        v, a, k = tree.lookup(torch.from_numpy(c.astype(np.int32)).to(_dev()))
        out = (v.cpu().numpy(), a.cpu().numpy().astype(bool))
        return out + (k.cpu().numpy(),) if with_kind else out
    finally:
        tree.close()
