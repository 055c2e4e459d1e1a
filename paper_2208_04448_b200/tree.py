"""Device upper tree: the flattened [Hash,5,4,3] tree for coordinate lookup.

Replaces ``VdbGrid.get_values(coords, with_kind=True)`` (grid.py:310-390)
with ``nvdb_lookup`` (csrc/lookup.cu).
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from ._lib import TreeDesc, check, lib
from .model import L1_SIZE, L2_SIZE, LEAF_SIZE, DenseLeafGrid


def _words(bits: np.ndarray, nbits: int) -> np.ndarray:
    """(n, nbits) bool -> (n, nbits/64) little-endian uint64 words (bit i = slot i)."""
    b = np.asarray(bits, dtype=bool).reshape(-1, nbits)
    packed = np.packbits(b, axis=1, bitorder="little")
    return np.ascontiguousarray(packed).view(np.uint64).reshape(b.shape[0], nbits // 64)


def tree_arrays(grid: DenseLeafGrid):
    """Host arrays of nvdb_tree_desc for a DenseLeafGrid (canonical order)."""
    l2o = np.asarray(grid.l2_origins, dtype=np.int64).reshape(-1, 3)
    l1o = np.asarray(grid.l1_origins, dtype=np.int64).reshape(-1, 3)
    # child bases: level-1 nodes are stored in (root, idx2) order and leaves
    # in (level-1 node, idx1) order, so bases are running sums of child counts
    n2c = grid.l2_child.reshape(-1, L2_SIZE).sum(axis=1)
    n1c = grid.l1_child.reshape(-1, L1_SIZE).sum(axis=1)
    l2_base = np.concatenate([[0], np.cumsum(n2c)[:-1]]).astype(np.int32) if len(n2c) else np.zeros(0, np.int32)
    l1_base = np.concatenate([[0], np.cumsum(n1c)[:-1]]).astype(np.int32) if len(n1c) else np.zeros(0, np.int32)
    if int(n2c.sum()) != l1o.shape[0] or int(n1c.sum()) != grid.leaf_origins.shape[0]:
        raise ValueError("grid child masks do not match node counts")
    roots = {}
    for i, o in enumerate(l2o):
        roots[tuple(int(v) for v in o)] = (i, 0.0, False)
    for k, (v, a) in grid.root_tiles.items():
        if tuple(k) not in roots:
            roots[tuple(int(x) for x in k)] = (-1, float(v), bool(a))
    keys = sorted(roots)
    return dict(
        root_keys=np.asarray(keys, dtype=np.int32).reshape(-1, 3),
        root_l2=np.asarray([roots[k][0] for k in keys], dtype=np.int32),
        root_tile_value=np.asarray([roots[k][1] for k in keys], dtype=np.float32),
        root_tile_active=np.asarray([roots[k][2] for k in keys], dtype=np.uint8),
        l2_child=_words(grid.l2_child, L2_SIZE), l2_active=_words(grid.l2_active, L2_SIZE),
        l2_tiles=np.ascontiguousarray(grid.l2_tiles, dtype=np.float32).reshape(-1, L2_SIZE),
        l2_child_base=l2_base,
        l1_child=_words(grid.l1_child, L1_SIZE), l1_active=_words(grid.l1_active, L1_SIZE),
        l1_tiles=np.ascontiguousarray(grid.l1_tiles, dtype=np.float32).reshape(-1, L1_SIZE),
        l1_child_base=l1_base,
        leaf_active=_words(grid.leaf_active, LEAF_SIZE),
        leaf_values=np.ascontiguousarray(grid.leaf_values, dtype=np.float32).reshape(-1, LEAF_SIZE),
    )


class DeviceTree:
    """Device-resident tree for ``nvdb_lookup``."""

    def __init__(self, grid: DenseLeafGrid):
        arr = tree_arrays(grid)
        self._keep = {k: np.ascontiguousarray(v) for k, v in arr.items()}
        p = lambda k: self._keep[k].ctypes.data_as(C.c_void_p)  # noqa: E731
        d = TreeDesc(background=float(grid.background), nroots=self._keep["root_keys"].shape[0],
                     n2=self._keep["l2_child"].shape[0], n1=self._keep["l1_child"].shape[0],
                     nl=self._keep["leaf_active"].shape[0],
                     root_keys=p("root_keys"), root_l2=p("root_l2"), root_tile_value=p("root_tile_value"),
                     root_tile_active=p("root_tile_active"), l2_child=p("l2_child"), l2_active=p("l2_active"),
                     l2_tiles=p("l2_tiles"), l2_child_base=p("l2_child_base"), l1_child=p("l1_child"),
                     l1_active=p("l1_active"), l1_tiles=p("l1_tiles"), l1_child_base=p("l1_child_base"),
                     leaf_active=p("leaf_active"), leaf_values=p("leaf_values"))
        h = C.c_void_p()
        check(lib().nvdb_tree_create(C.byref(d), C.byref(h)), "nvdb_tree_create")
        self.handle = h
        del self._keep

    def close(self) -> None:
        if getattr(self, "handle", None) is not None and self.handle.value:
            lib().nvdb_tree_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass

    def lookup(self, coords: torch.Tensor, want_leaf: bool = False):
        """(value f32, active u8, kind u8[, leaf i32]) for int32 device coords (n,3)."""
        assert coords.is_cuda and coords.dtype == torch.int32 and coords.is_contiguous()
        n = coords.shape[0]
        dev = coords.device
        val = torch.empty(n, dtype=torch.float32, device=dev)
        act = torch.empty(n, dtype=torch.uint8, device=dev)
        kind = torch.empty(n, dtype=torch.uint8, device=dev)
        leaf = torch.empty(n, dtype=torch.int32, device=dev) if want_leaf else None
        check(lib().nvdb_lookup(self.handle, coords.data_ptr(), n, val.data_ptr(), act.data_ptr(),
                                kind.data_ptr(), leaf.data_ptr() if leaf is not None else None,
                                torch.cuda.current_stream(dev).cuda_stream), "nvdb_lookup")
        return (val, act, kind, leaf) if want_leaf else (val, act, kind)
