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

    def __init__(self, grid: DenseLeafGrid = None, arrays=None, background: float = 0.0):
        if grid is not None:
            arrays = tree_arrays(grid)
            background = float(grid.background)
        keep = {}
        for k, v in arrays.items():
            keep[k] = v.contiguous() if isinstance(v, torch.Tensor) else np.ascontiguousarray(v)

        def p(k):
            v = keep.get(k)
            if v is None:
                return None
            return v.data_ptr() if isinstance(v, torch.Tensor) else v.ctypes.data_as(C.c_void_p)

        def rows(k, w):
            v = keep[k]
            return int(v.numel() // w) if isinstance(v, torch.Tensor) else int(v.size // w)

        d = TreeDesc(background=float(background), nroots=rows("root_l2", 1), n2=rows("l2_child", 512),
                     n1=rows("l1_child", 64), nl=rows("leaf_active", 8),
                     root_keys=p("root_keys"), root_l2=p("root_l2"), root_tile_value=p("root_tile_value"),
                     root_tile_active=p("root_tile_active"), l2_child=p("l2_child"), l2_active=p("l2_active"),
                     l2_tiles=p("l2_tiles"), l2_child_base=p("l2_child_base"), l1_child=p("l1_child"),
                     l1_active=p("l1_active"), l1_tiles=p("l1_tiles"), l1_child_base=p("l1_child_base"),
                     leaf_active=p("leaf_active"), leaf_values=p("leaf_values"),
                     leaf_patched=p("leaf_patched"))
        torch.cuda.synchronize()
        h = C.c_void_p()
        check(lib().nvdb_tree_create(C.byref(d), C.byref(h)), "nvdb_tree_create")
        self.handle = h

    @classmethod
    def from_decode(cls, d) -> "DeviceTree":
        """Hybrid topology of a device decode (decoder.py:52-81 + _fill_leaves wiring)."""
        from ._lib import lib as _l  # noqa: WPS433
        d.check()
        m = d.model
        c = m.c
        ut = c.upper_tree
        dev = m.dev
        st = torch.cuda.current_stream(dev).cuda_stream
        n1 = m.n1
        # level-2 nodes and roots from the container (explicit)
        l2o = np.asarray([n.origin for n in ut.l2_nodes], dtype=np.int64).reshape(-1, 3)
        o2 = np.lexsort((l2o[:, 2], l2o[:, 1], l2o[:, 0])) if len(l2o) else np.zeros(0, np.int64)
        bg = np.float32(c.grid_meta.background)
        l2c = np.zeros((len(o2), L2_SIZE), bool)
        l2a = np.zeros((len(o2), L2_SIZE), bool)
        l2t = np.full((len(o2), L2_SIZE), bg, np.float32)
        for j, i in enumerate(o2):
            nd = ut.l2_nodes[i]
            l2c[j] = nd.child_mask.bits
            l2a[j] = nd.active_mask.bits
            for k, v in nd.tiles.items():
                l2t[j, int(k)] = v
        n2c = l2c.sum(axis=1)
        l2_base = (np.concatenate([[0], np.cumsum(n2c)[:-1]]) if len(n2c) else np.zeros(0)).astype(np.int32)
        roots = {tuple(int(v) for v in l2o[i]): (j, 0.0, False) for j, i in enumerate(o2)}
        for k, (v, a) in ut.root_tiles.items():
            roots.setdefault(tuple(int(x) for x in k), (-1, float(v), bool(a)))
        keys = sorted(roots)
        # level-1 nodes in tree order (root-major), leaves stay in decode order
        rk = m.origins & ~np.int64(4095)
        order = np.lexsort((m.origins[:, 2], m.origins[:, 1], m.origins[:, 0], rk[:, 2], rk[:, 1], rk[:, 0])) \
            if n1 else np.zeros(0, np.int64)
        order_t = torch.from_numpy(order.astype(np.int64)).to(dev)
        cls2 = d.l1_class.view(max(n1, 1), L1_SIZE) if n1 else d.l1_class.view(0, L1_SIZE)
        counts = (cls2 == 0).sum(dim=1)
        starts = torch.cumsum(counts, 0) - counts
        cw = torch.empty((max(n1, 1) * 64,), dtype=torch.int64, device=dev)
        aw = torch.empty((max(n1, 1) * 64,), dtype=torch.int64, device=dev)
        check(_l().nvdb_pack_eq(d.l1_class.data_ptr(), n1 * 64, 0, cw.data_ptr(), st), "pack child")
        check(_l().nvdb_pack_eq(d.l1_class.data_ptr(), n1 * 64, 1, aw.data_ptr(), st), "pack active")
        nl = d.leaf_count
        pw = torch.empty((max(nl, 1) * 8,), dtype=torch.int64, device=dev)
        check(_l().nvdb_pack_eq(d.patched.data_ptr(), nl * 8, 1, pw.data_ptr(), st), "pack patched")
        arrays = dict(
            root_keys=np.asarray(keys, dtype=np.int32).reshape(-1, 3),
            root_l2=np.asarray([roots[k][0] for k in keys], dtype=np.int32),
            root_tile_value=np.asarray([roots[k][1] for k in keys], dtype=np.float32),
            root_tile_active=np.asarray([roots[k][2] for k in keys], dtype=np.uint8),
            l2_child=_words(l2c, L2_SIZE), l2_active=_words(l2a, L2_SIZE), l2_tiles=l2t,
            l2_child_base=l2_base,
            l1_child=cw[:n1 * 64].view(n1, 64)[order_t] if n1 else cw[:0],
            l1_active=aw[:n1 * 64].view(n1, 64)[order_t] if n1 else aw[:0],
            l1_tiles=d.l1_tiles.view(n1, L1_SIZE)[order_t] if n1 else d.l1_tiles[:0],
            l1_child_base=starts[order_t].to(torch.int32) if n1 else torch.zeros(0, dtype=torch.int32, device=dev),
            leaf_active=d.active_words[:nl * 8], leaf_values=d.leaf_values[:nl * 512],
            leaf_patched=pw[:nl * 8],
        )
        return cls(arrays=arrays, background=float(bg))

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

    def lookup_rows(self, coords: torch.Tensor):
        """lookup() fused with the query's neural-row selection
        (nvdb_lookup_rows): (value, active, kind, rows, count, npatched);
        rows[:count] are the active leaf-voxel rows without an exact patch
        (device int64 count), npatched the active leaf-voxel rows answered
        by a patch."""
        assert coords.is_cuda and coords.dtype == torch.int32 and coords.is_contiguous()
        n = coords.shape[0]
        dev = coords.device
        val = torch.empty(n, dtype=torch.float32, device=dev)
        act = torch.empty(n, dtype=torch.uint8, device=dev)
        kind = torch.empty(n, dtype=torch.uint8, device=dev)
        rows = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
        cnt = torch.empty(2, dtype=torch.int64, device=dev)
        check(lib().nvdb_lookup_rows(self.handle, coords.data_ptr(), n, val.data_ptr(), act.data_ptr(),
                                     kind.data_ptr(), rows.data_ptr(), cnt.data_ptr(), cnt[1:].data_ptr(),
                                     torch.cuda.current_stream(dev).cuda_stream), "nvdb_lookup_rows")
        return val, act, kind, rows, cnt[:1], cnt[1:]
