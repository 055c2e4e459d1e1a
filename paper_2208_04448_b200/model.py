"""Host-side data model for the NeuralVDB hot path.

The classes mirror the attribute names of the reference package's
``svcodec`` types (``container.py:62-153``, ``neural.py:37-165``,
``partition.py:25-71``) so code written against either works with both
(duck typing): a ``NeuralGridContainer`` decoded by the reference can be
handed to :func:`paper_2208_04448_b200.decode_full` unchanged, and the
containers this package produces expose the same fields.

The explicit grid is held as a :class:`DenseLeafGrid`: flat arrays of
level-2 nodes, level-1 nodes and dense 8^3 leaves (the reference's
``VdbGrid`` object tree, ``grid.py:248-390``, flattened).  Converters to
and from ``svcodec`` objects are provided for interop; they are plain host
plumbing and never on the hot path.
"""

from __future__ import annotations

import itertools
from collections.abc import MutableMapping
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Tuple

import numpy as np

Coord = Tuple[int, int, int]

LEAF_LOG2, L1_LOG2, L2_LOG2 = 3, 4, 5
LEAF_SPAN = 8
L1_SPAN = 128
L2_SPAN = 4096
LEAF_SIZE = 512
L1_SIZE = 4096
L2_SIZE = 32768

L1_CLASS_CHILD = 0          # container.py:57
L1_CLASS_ACTIVE_TILE = 1    # container.py:58
L1_CLASS_INACTIVE_TILE = 2  # container.py:59

GRID_CLASS_SDF = "sdf"
GRID_CLASS_FOG = "fog"
HALO = 8                    # partition.py:21
NET_TAGS = {"l1": 0, "tile": 1, "l0": 2, "voxel": 3}   # encoder.py:86


def local_coords(log2dim: int) -> np.ndarray:
    """(8^L, 3) slot offsets in index order (x major, z fastest; grid.py:48-52)."""
    n = 1 << log2dim
    idx = np.arange(n ** 3)
    return np.stack([idx >> (2 * log2dim), (idx >> log2dim) & (n - 1), idx & (n - 1)],
                    axis=1).astype(np.int64)


LEAF_LOCAL = local_coords(LEAF_LOG2)
L1_LOCAL = local_coords(L1_LOG2)


# -- networks -------------------------------------------------------------------


@dataclass
class Activation:
    kind: str = "relu"
    frequency: float = 1.0


class FourierFeatures:
    """Gaussian frequency matrix regenerated from (seed, m, scale) (neural.py:51-69)."""

    def __init__(self, m: int, scale: float, seed: int, amplitude: float = 1.0):
        self.m = int(m)
        self.scale = float(scale)
        self.seed = int(seed)
        self.amplitude = float(amplitude)
        self.matrix = np.random.default_rng(self.seed).standard_normal((self.m, 3)) * self.scale

    @property
    def out_dim(self) -> int:
        return 2 * self.m


class MlpParams:
    def __init__(self, layers, activation: Activation, head: str = "linear"):
        self.layers = layers
        self.activation = activation
        self.head = head

    @property
    def in_dim(self) -> int:
        return self.layers[0][0].shape[1]

    @property
    def out_dim(self) -> int:
        return self.layers[-1][0].shape[0]

    @property
    def dims(self) -> List[int]:
        return [self.in_dim] + [w.shape[0] for w, _ in self.layers]

    def copy(self) -> "MlpParams":
        return MlpParams([(w.copy(), b.copy()) for w, b in self.layers],
                         Activation(self.activation.kind, self.activation.frequency),
                         self.head)

    def parameter_count(self) -> int:
        return sum(w.size + b.size for w, b in self.layers)

    def flatten(self) -> np.ndarray:
        """All parameters, layer by layer, weights then bias (neural.py:164-165)."""
        return np.concatenate([np.concatenate([w.ravel(), b.ravel()]) for w, b in self.layers])


@dataclass
class NetRecord:
    params: MlpParams
    ff: FourierFeatures
    final_loss: float = 0.0
    epochs: int = 0


# -- layout ---------------------------------------------------------------------


@dataclass
class Subdomain:
    id: int
    cell: Coord
    size: int
    cluster_id: int = 0
    halo: int = HALO

    @property
    def lo(self) -> np.ndarray:
        return np.asarray(self.cell, dtype=np.int64) * self.size

    @property
    def hi(self) -> np.ndarray:
        return self.lo + self.size

    def expanded_lo(self) -> np.ndarray:
        return self.lo - self.halo

    def expanded_hi(self) -> np.ndarray:
        return self.hi + self.halo


@dataclass
class SubdomainLayout:
    size: int
    halo: int = HALO
    subdomains: List[Subdomain] = field(default_factory=list)
    cell_to_id: Dict[Coord, int] = field(default_factory=dict)
    cluster_count: int = 0


# -- container --------------------------------------------------------------------


class Mask:
    """Bit container with the ``.bits`` attribute of svcodec's NodeMask."""

    def __init__(self, bits):
        self.bits = np.asarray(bits, dtype=bool)

    def indices(self) -> np.ndarray:
        return np.flatnonzero(self.bits)

    def count(self) -> int:
        return int(np.count_nonzero(self.bits))

    def packed_words(self) -> bytes:
        """grid.py:167-169: little-endian packed bits (container serialization)."""
        return np.packbits(self.bits, bitorder="little").tobytes()


@dataclass
class GridMeta:
    grid_class: str
    background: float
    voxel_size: float
    half_width: float
    value_scale: float


@dataclass
class L2NodeRecord:
    origin: Coord
    child_mask: Mask
    active_mask: Mask
    tiles: Dict[int, float] = field(default_factory=dict)


class LeafBitsMap(MutableMapping):
    """Array-backed ``{leaf origin: (512,) bool}`` (the reference's
    ``UpperTree.leaf_negative_fill`` dict, container.py / encoder.py:519-526):
    a mapping for lookups, iteration and assignment that hands the decoder its
    (n, 3) origins and (n, 512) bits without a per-leaf conversion."""

    def __init__(self, items=None):
        self._keys = np.zeros((0, 3), np.int64)
        self._bits = np.zeros((0, LEAF_SIZE), bool)
        self._index = None  # origin tuple -> row, built on first keyed access
        self._extra = {}    # keys assigned one by one, merged on arrays()
        if items:
            for k, v in (items.items() if hasattr(items, "items") else items):
                self[k] = v

    @classmethod
    def from_arrays(cls, keys, bits) -> "LeafBitsMap":
        m = cls()
        keys = np.asarray(keys, np.int64).reshape(-1, 3)
        bits = np.asarray(bits, bool).reshape(-1, LEAF_SIZE)
        if keys.shape[0] != bits.shape[0]:
            raise ValueError("leaf origins and bit rows differ in count")
        if keys.shape[0] and np.unique(keys, axis=0).shape[0] != keys.shape[0]:
            raise ValueError("duplicate leaf origins")
        m._keys, m._bits = keys.copy(), bits.copy()
        return m

    def arrays(self):
        """(origins (n, 3) int64, bits (n, 512) bool) in insertion order."""
        if self._extra:
            n0 = self._keys.shape[0]
            ks = np.asarray(list(self._extra.keys()), np.int64).reshape(-1, 3)
            bs = np.stack(list(self._extra.values()))
            self._keys = np.concatenate([self._keys, ks])
            self._bits = np.concatenate([self._bits, bs])
            if self._index is not None:
                self._index.update((k, n0 + i) for i, k in enumerate(self._extra))
            self._extra = {}
        return self._keys, self._bits

    def _row(self, key):
        """Row of an origin in the arrays (extras not included), or None."""
        if self._index is None:
            self._index = {tuple(int(v) for v in k): i for i, k in enumerate(self._keys)}
        return self._index.get(key)

    def __getitem__(self, key):
        key = tuple(int(v) for v in key)
        if key in self._extra:
            return self._extra[key]
        i = self._row(key)
        if i is None:
            raise KeyError(key)
        return self._bits[i]

    def __setitem__(self, key, value):
        key = tuple(int(v) for v in key)
        v = np.asarray(value, bool).reshape(LEAF_SIZE)
        i = self._row(key) if self._keys.shape[0] and key not in self._extra else None
        if i is None:
            self._extra[key] = v
        else:
            self._bits[i] = v

    def __delitem__(self, key):
        key = tuple(int(v) for v in key)
        if key in self._extra:
            del self._extra[key]
            return
        i = self._row(key)
        if i is None:
            raise KeyError(key)
        self._keys = np.delete(self._keys, i, axis=0)
        self._bits = np.delete(self._bits, i, axis=0)
        self._index = None

    def __iter__(self):
        self.arrays()
        return (tuple(int(v) for v in k) for k in self._keys)

    def __len__(self) -> int:
        return self._keys.shape[0] + len(self._extra)

    def __repr__(self) -> str:
        return f"LeafBitsMap(n={len(self)})"

    def __getstate__(self):
        k, b = self.arrays()
        return (k, np.packbits(b, axis=1, bitorder="little"))

    def __setstate__(self, st):
        self._keys = st[0]
        self._bits = np.unpackbits(st[1], axis=1, count=LEAF_SIZE, bitorder="little").astype(bool)
        self._index, self._extra = None, {}


class L1TileMap(MutableMapping):
    """Array-backed ``{level-1 node origin: {slot: tile value}}`` (the
    reference's ``UpperTree.l1_tiles`` dict of dicts, encoder.py:512-517): a
    mapping for the reference's readers (container writer, decoder loops) that
    hands the device decode its records as columns without a per-record
    conversion.  Rows are grouped per node in insertion order."""

    def __init__(self, items=None):
        self._org = np.zeros((0, 3), np.int64)
        self._cnt = np.zeros(0, np.int64)
        self._slot = np.zeros(0, np.int64)
        self._val = np.zeros(0, np.float32)
        self._extra = {}  # nodes assigned one by one (merged on arrays())
        if items:
            for k, v in (items.items() if hasattr(items, "items") else items):
                self[k] = v

    @classmethod
    def from_arrays(cls, node_origins, counts, slots, values) -> "L1TileMap":
        m = cls()
        m._org = np.asarray(node_origins, np.int64).reshape(-1, 3).copy()
        m._cnt = np.asarray(counts, np.int64).reshape(-1).copy()
        m._slot = np.asarray(slots, np.int64).reshape(-1).copy()
        m._val = np.asarray(values, np.float32).reshape(-1).copy()
        if m._org.shape[0] != m._cnt.shape[0] or int(m._cnt.sum()) != m._slot.shape[0] != m._val.shape[0]:
            raise ValueError("tile map columns disagree")
        return m

    def arrays(self):
        """(node origins (k, 3), records per node (k,), slots (n,), values (n,))."""
        if self._extra:
            org = [self._org] + [np.asarray([k], np.int64) for k in self._extra]
            cnt = [self._cnt] + [np.asarray([len(d)], np.int64) for d in self._extra.values()]
            sl = [self._slot] + [np.fromiter(d.keys(), np.int64, len(d)) for d in self._extra.values()]
            vl = [self._val] + [np.fromiter(d.values(), np.float32, len(d)) for d in self._extra.values()]
            self._org, self._cnt = np.concatenate(org), np.concatenate(cnt)
            self._slot, self._val = np.concatenate(sl), np.concatenate(vl)
            self._extra = {}
        return self._org, self._cnt, self._slot, self._val

    def _rows(self):
        return {tuple(int(v) for v in o): i for i, o in enumerate(self._org)}

    def __getitem__(self, key):
        key = tuple(int(v) for v in key)
        if key in self._extra:
            return self._extra[key]
        i = self._rows().get(key)
        if i is None:
            raise KeyError(key)
        s = int(self._cnt[:i].sum())
        e = s + int(self._cnt[i])
        return dict(zip(self._slot[s:e].tolist(), self._val[s:e].astype(np.float64).tolist()))

    def __setitem__(self, key, value):
        key = tuple(int(v) for v in key)
        if key in self._rows():
            del self[key]
        self._extra[key] = {int(k): float(v) for k, v in dict(value).items()}

    def __delitem__(self, key):
        key = tuple(int(v) for v in key)
        if key in self._extra:
            del self._extra[key]
            return
        i = self._rows().get(key)
        if i is None:
            raise KeyError(key)
        s = int(self._cnt[:i].sum())
        e = s + int(self._cnt[i])
        self._org = np.delete(self._org, i, axis=0)
        self._cnt = np.delete(self._cnt, i)
        self._slot = np.delete(self._slot, np.s_[s:e])
        self._val = np.delete(self._val, np.s_[s:e])

    def __iter__(self):
        self.arrays()
        return (tuple(int(v) for v in o) for o in self._org)

    def __len__(self) -> int:
        return self._org.shape[0] + len(self._extra)

    def __repr__(self) -> str:
        return f"L1TileMap(nodes={len(self)}, records={int(self._cnt.sum())})"

    def __getstate__(self):
        return self.arrays()

    def __setstate__(self, st):
        self._org, self._cnt, self._slot, self._val = st
        self._extra = {}


@dataclass
class UpperTree:
    root_tiles: Dict[Coord, Tuple[float, bool]] = field(default_factory=dict)
    l2_nodes: List[L2NodeRecord] = field(default_factory=list)
    l1_origins: List[Coord] = field(default_factory=list)
    l1_tiles: Dict[Coord, Dict[int, float]] = field(default_factory=dict)
    leaf_negative_fill: LeafBitsMap = field(default_factory=LeafBitsMap)


class PatchRecords:
    """Array-backed list of patch records (container.py:100-117 keeps Python
    lists of tuples): level-1 records ``(origin, cls)``, level-0 records
    ``(coord, active, value)``.  Behaves as the reference's list for
    ``append`` / iteration / indexing / ``len`` / ``==``, and hands the decoder
    its columns without a per-record conversion (:meth:`arrays`)."""

    __slots__ = ("level", "_keys", "_cols", "_pending")

    def __init__(self, level: int, records=()):
        self.level = int(level)
        self._keys = np.zeros((0, 3), np.int64)
        self._cols = [np.zeros(0, np.int64)] if self.level == 1 else [np.zeros(0, bool), np.zeros(0, np.float64)]
        self._pending = []
        for r in records:
            self.append(r)

    def append(self, rec) -> None:
        self._pending.append(rec)

    def extend_arrays(self, keys, *cols) -> None:
        """Append records given as columns: keys (n, 3) and the record's fields."""
        self._flush()
        keys = np.asarray(keys, np.int64).reshape(-1, 3)
        if len(cols) != len(self._cols) or any(np.shape(c) != (keys.shape[0],) for c in cols):
            raise ValueError("patch columns do not match the record layout")
        self._keys = np.concatenate([self._keys, keys])
        self._cols = [np.concatenate([a, np.asarray(c, a.dtype)]) for a, c in zip(self._cols, cols)]

    def _flush(self) -> None:
        if not self._pending:
            return
        lst, self._pending = self._pending, []
        n = len(lst)
        cols = list(zip(*lst))
        keys = np.fromiter(itertools.chain.from_iterable(cols[0]), dtype=np.int64, count=3 * n).reshape(-1, 3)
        self._keys = np.concatenate([self._keys, keys])
        self._cols = [np.concatenate([a, np.fromiter(c, dtype=a.dtype, count=n)]) for a, c in zip(self._cols, cols[1:])]

    def arrays(self):
        """(keys (n, 3) int64, *columns): l1 -> (cls int64,), l0 -> (active bool, value float64)."""
        self._flush()
        return (self._keys, *self._cols)

    def __len__(self) -> int:
        return self._keys.shape[0] + len(self._pending)

    def _record(self, i: int):
        k = tuple(int(v) for v in self._keys[i])
        if self.level == 1:
            return (k, int(self._cols[0][i]))
        return (k, bool(self._cols[0][i]), float(self._cols[1][i]))

    def __getitem__(self, i):
        self._flush()
        if isinstance(i, slice):
            return [self._record(j) for j in range(*i.indices(len(self)))]
        n = len(self)
        if not -n <= i < n:
            raise IndexError("patch index out of range")
        return self._record(i % n)

    def __iter__(self):
        self._flush()
        return (self._record(i) for i in range(len(self)))

    def __eq__(self, other) -> bool:
        try:
            return len(self) == len(other) and all(a == b for a, b in zip(self, other))
        except TypeError:
            return NotImplemented

    def __repr__(self) -> str:
        return f"PatchRecords(level={self.level}, n={len(self)})"

    def __getstate__(self):
        self._flush()
        return (self.level, self._keys, self._cols)

    def __setstate__(self, st):
        self.level, self._keys, self._cols = st
        self._pending = []


def _patch_records(level: int, records):
    if isinstance(records, PatchRecords):
        return records
    return PatchRecords(level, records)


@dataclass
class PatchList:
    l1: PatchRecords = field(default_factory=lambda: PatchRecords(1))
    l0: PatchRecords = field(default_factory=lambda: PatchRecords(0))

    def __post_init__(self):
        self.l1 = _patch_records(1, self.l1)
        self.l0 = _patch_records(0, self.l0)

    def __len__(self) -> int:
        return len(self.l1) + len(self.l0)


@dataclass
class EncodedSubdomain:
    id: int
    cell: Coord
    cluster_id: int
    norm_origin: np.ndarray
    norm_scale: float
    value_scale: float
    l1_classifier: Optional[NetRecord] = None
    tile_regressor: Optional[NetRecord] = None
    l0_classifier: Optional[NetRecord] = None
    voxel_regressor: Optional[NetRecord] = None
    patches: PatchList = field(default_factory=PatchList)

    def nets(self):
        return [("l1", self.l1_classifier), ("tile", self.tile_regressor),
                ("l0", self.l0_classifier), ("voxel", self.voxel_regressor)]


@dataclass
class NeuralGridContainer:
    grid_meta: GridMeta
    upper_tree: UpperTree
    layout: SubdomainLayout
    experts: List[EncodedSubdomain]
    config: object = None
    weight_precision: int = 32

    def payload_bytes(self) -> int:
        """container.py:167-169 (svcodec's own payload builder)."""
        from svcodec.container import _build_payload  # noqa: WPS433
        return len(_build_payload(self))

    def parameter_count(self) -> int:
        return sum(n.params.parameter_count() for e in self.experts for _, n in e.nets() if n is not None)

    def patch_count(self) -> int:
        return sum(len(e.patches) for e in self.experts)


# -- explicit grid ----------------------------------------------------------------


@dataclass
class DenseLeafGrid:
    """Flattened [Hash,5,4,3] tree (grid.py:248-390 as arrays).

    Ordering: level-2 nodes by sorted root key; level-1 nodes and leaves in
    canonical (root key, idx2, idx1) order, i.e. the order of
    ``VdbGrid.iter_leaves`` (grid.py:397-404).
    """

    background: float
    grid_class: str
    voxel_size: float
    half_width: float
    root_tiles: Dict[Coord, Tuple[float, bool]]
    l2_origins: np.ndarray     # (n2, 3) int64
    l2_child: np.ndarray       # (n2, 32768) bool
    l2_active: np.ndarray      # (n2, 32768) bool
    l2_tiles: np.ndarray       # (n2, 32768) f32
    l1_origins: np.ndarray     # (n1, 3) int64
    l1_child: np.ndarray       # (n1, 4096) bool
    l1_active: np.ndarray      # (n1, 4096) bool
    l1_tiles: np.ndarray       # (n1, 4096) f32
    leaf_origins: np.ndarray   # (nl, 3) int64
    leaf_active: np.ndarray    # (nl, 512) bool
    leaf_values: np.ndarray    # (nl, 512) f32

    @property
    def leaf_count(self) -> int:
        return int(self.leaf_origins.shape[0])

    def active_voxel_count(self) -> int:
        return int(self.leaf_active.sum())

    def active_voxels(self):
        """(coords, values) of active leaf voxels in canonical order."""
        li, vi = np.nonzero(self.leaf_active)
        coords = self.leaf_origins[li] + LEAF_LOCAL[vi]
        return coords, self.leaf_values[li, vi]

    def active_tiles(self):
        """(origin, extent) of active tiles at every level (decompose input)."""
        out = []
        for key, (_, act) in sorted(self.root_tiles.items()):
            if act:
                out.append((key, L2_SPAN))
        for ni in range(self.l2_origins.shape[0]):
            for idx in np.flatnonzero(self.l2_active[ni] & ~self.l2_child[ni]):
                out.append((tuple(int(v) for v in self.l2_origins[ni] + L1_SPAN * local_coords(L2_LOG2)[idx]), L1_SPAN))
        for ni in range(self.l1_origins.shape[0]):
            for idx in np.flatnonzero(self.l1_active[ni] & ~self.l1_child[ni]):
                out.append((tuple(int(v) for v in self.l1_origins[ni] + LEAF_SPAN * L1_LOCAL[idx]), LEAF_SPAN))
        return out

    # -- interop ----------------------------------------------------------------

    @classmethod
    def from_svcodec(cls, grid) -> "DenseLeafGrid":
        """Flatten an svcodec ``VdbGrid`` (walks its node objects once)."""
        l2o, l2c, l2a, l2t = [], [], [], []
        l1o, l1c, l1a, l1t = [], [], [], []
        lo, la, lv = [], [], []
        for key in sorted(grid.root):
            n2 = grid.root[key]
            l2o.append(key)
            l2c.append(n2.child_mask.bits.copy())
            l2a.append(n2.active_mask.bits.copy())
            l2t.append(np.asarray(n2.tiles, dtype=np.float32).copy())
            for idx2 in np.flatnonzero(n2.child_mask.bits):
                n1 = n2.children[int(idx2)]
                l1o.append(n1.origin)
                l1c.append(n1.child_mask.bits.copy())
                l1a.append(n1.active_mask.bits.copy())
                l1t.append(np.asarray(n1.tiles, dtype=np.float32).copy())
                for idx1 in np.flatnonzero(n1.child_mask.bits):
                    leaf = n1.children[int(idx1)]
                    lo.append(leaf.origin)
                    la.append(leaf.active.bits.copy())
                    lv.append(np.asarray(leaf.values, dtype=np.float32).copy())

        def st(rows, dtype, width):
            return np.asarray(rows, dtype=dtype) if rows else np.zeros((0, width), dtype=dtype)

        return cls(
            background=float(grid.background), grid_class=grid.grid_class,
            voxel_size=float(grid.voxel_size), half_width=float(grid.half_width),
            root_tiles=dict(grid.root_tiles),
            l2_origins=st(l2o, np.int64, 3), l2_child=st(l2c, bool, L2_SIZE),
            l2_active=st(l2a, bool, L2_SIZE), l2_tiles=st(l2t, np.float32, L2_SIZE),
            l1_origins=st(l1o, np.int64, 3), l1_child=st(l1c, bool, L1_SIZE),
            l1_active=st(l1a, bool, L1_SIZE), l1_tiles=st(l1t, np.float32, L1_SIZE),
            leaf_origins=st(lo, np.int64, 3), leaf_active=st(la, bool, LEAF_SIZE),
            leaf_values=st(lv, np.float32, LEAF_SIZE),
        )

    def to_svcodec(self):
        """Rebuild an svcodec ``VdbGrid`` (requires the reference package).

        Vectorized assembly (decoder.py:197-210): node
        masks, tiles and leaf values are row views of this grid's dense
        arrays (copied once into contiguous blocks owned by the new grid), and
        the node objects are created without their constructors' per-node
        ``np.full`` / mask allocation, so the host cost is one small object
        per node instead of three 512- to 32768-element array allocations."""
        from svcodec.grid import InternalNode, LeafNode, NodeMask, VdbGrid  # noqa: WPS433
        g = VdbGrid(self.background, self.grid_class, self.voxel_size, self.half_width)
        g.root_tiles = dict(self.root_tiles)
        new_leaf, new_node, new_mask = LeafNode.__new__, InternalNode.__new__, NodeMask.__new__

        def mask(bits):
            mk = new_mask(NodeMask)
            mk.bits = bits
            return mk

        def node(origin, log2dim, child, active, tiles):
            n = new_node(InternalNode)
            n.origin = origin
            n.log2dim = log2dim
            n.slot_span = (LEAF_SPAN << log2dim if log2dim == L1_LOG2 else L1_SPAN << log2dim) >> log2dim
            n.child_mask = mask(child)
            n.active_mask = mask(active)
            n.tiles = tiles
            n.children = {}
            return n

        n2 = self.l2_origins.shape[0]
        c2, a2 = np.array(self.l2_child, dtype=bool), np.array(self.l2_active, dtype=bool)
        t2 = np.array(self.l2_tiles, dtype=np.float32)
        for ni, key in enumerate(map(tuple, self.l2_origins.tolist())):
            g.root[key] = node(key, L2_LOG2, c2[ni], a2[ni], t2[ni])
        n1 = self.l1_origins.shape[0]
        c1, a1 = np.array(self.l1_child, dtype=bool), np.array(self.l1_active, dtype=bool)
        t1 = np.array(self.l1_tiles, dtype=np.float32)
        o1 = self.l1_origins.astype(np.int64)
        roots1 = map(tuple, (o1 & ~np.int64(L2_SPAN - 1)).tolist())
        idx2 = ((((o1[:, 0] & 4095) >> 7) << 10) | (((o1[:, 1] & 4095) >> 7) << 5) | ((o1[:, 2] & 4095) >> 7)).tolist()
        l1_nodes = []
        for ni, (org, root, k2) in enumerate(zip(map(tuple, o1.tolist()), roots1, idx2)):
            nd = node(org, L1_LOG2, c1[ni], a1[ni], t1[ni])
            g.root[root].children[k2] = nd
            l1_nodes.append(nd)
        nl = self.leaf_origins.shape[0]
        if nl:
            la = np.array(self.leaf_active, dtype=bool).reshape(nl, LEAF_SIZE)
            lv = np.array(self.leaf_values, dtype=np.float32).reshape(nl, LEAF_SIZE)
            ol = self.leaf_origins.astype(np.int64)
            by_origin = dict(zip(map(tuple, o1.tolist()), l1_nodes))
            parents = map(tuple, (ol & ~np.int64(L1_SPAN - 1)).tolist())
            idx1 = ((((ol[:, 0] & 127) >> 3) << 8) | (((ol[:, 1] & 127) >> 3) << 4) | ((ol[:, 2] & 127) >> 3)).tolist()
            for li, (org, par, k1) in enumerate(zip(map(tuple, ol.tolist()), parents, idx1)):
                leaf = new_leaf(LeafNode)
                leaf.origin = org
                leaf.values = lv[li]
                leaf.active = mask(la[li])
                by_origin[par].children[k1] = leaf
        return g


# -- svcodec container interop -----------------------------------------------------


def _net_from_any(rec) -> Optional[NetRecord]:
    if rec is None:
        return None
    p = rec.params
    act = Activation(p.activation.kind, float(p.activation.frequency))
    layers = [(np.asarray(w, dtype=np.float32).copy(), np.asarray(b, dtype=np.float32).copy())
              for w, b in p.layers]
    ff = FourierFeatures(rec.ff.m, rec.ff.scale, rec.ff.seed, rec.ff.amplitude)
    return NetRecord(MlpParams(layers, act, p.head), ff, float(rec.final_loss), int(rec.epochs))


def container_from_any(c) -> NeuralGridContainer:
    """Copy any container exposing svcodec's attribute names into this model."""
    m = c.grid_meta
    meta = GridMeta(m.grid_class, float(m.background), float(m.voxel_size),
                    float(m.half_width), float(m.value_scale))
    ut = c.upper_tree
    tree = UpperTree(
        root_tiles={tuple(k): (float(v[0]), bool(v[1])) for k, v in ut.root_tiles.items()},
        l2_nodes=[L2NodeRecord(tuple(n.origin), Mask(n.child_mask.bits.copy()),
                               Mask(n.active_mask.bits.copy()), dict(n.tiles))
                  for n in ut.l2_nodes],
        l1_origins=[tuple(int(v) for v in o) for o in ut.l1_origins],
        l1_tiles={tuple(k): dict(v) for k, v in ut.l1_tiles.items()},
        leaf_negative_fill=_copy_leaf_bits(ut.leaf_negative_fill),
    )
    lay = c.layout
    layout = SubdomainLayout(size=int(lay.size), halo=int(lay.halo),
                             cluster_count=int(lay.cluster_count))
    for s in lay.subdomains:
        layout.subdomains.append(Subdomain(int(s.id), tuple(int(v) for v in s.cell),
                                           int(s.size), int(s.cluster_id), int(s.halo)))
        layout.cell_to_id[tuple(int(v) for v in s.cell)] = int(s.id)
    experts = []
    for e in c.experts:
        ex = EncodedSubdomain(
            id=int(e.id), cell=tuple(int(v) for v in e.cell), cluster_id=int(e.cluster_id),
            norm_origin=np.asarray(e.norm_origin, dtype=np.float64).copy(),
            norm_scale=float(e.norm_scale), value_scale=float(e.value_scale),
            l1_classifier=_net_from_any(e.l1_classifier),
            tile_regressor=_net_from_any(e.tile_regressor),
            l0_classifier=_net_from_any(e.l0_classifier),
            voxel_regressor=_net_from_any(e.voxel_regressor),
            patches=_copy_patches(e.patches),
        )
        experts.append(ex)
    return NeuralGridContainer(meta, tree, layout, experts, getattr(c, "config", None),
                               int(getattr(c, "weight_precision", 32)))


# -- npz fixtures (tests/golden) -----------------------------------------------------

_ACT = {"relu": 0, "tanh": 1, "sine": 2}
_HEAD = {"linear": 0, "logits": 1, "binary": 2}
_INV_ACT = {v: k for k, v in _ACT.items()}
_INV_HEAD = {v: k for k, v in _HEAD.items()}


def container_to_arrays(c, prefix: str = "c_") -> Dict[str, np.ndarray]:
    """Flatten a container into named arrays (for committed golden fixtures)."""
    c = container_from_any(c)
    a: Dict[str, np.ndarray] = {}
    m = c.grid_meta
    a["meta"] = np.array([0 if m.grid_class == GRID_CLASS_SDF else 1, m.background,
                          m.voxel_size, m.half_width, m.value_scale], dtype=np.float64)
    ut = c.upper_tree
    rk = sorted(ut.root_tiles)
    a["rt_origin"] = np.asarray(rk, dtype=np.int64).reshape(-1, 3)
    a["rt_value"] = np.asarray([ut.root_tiles[k][0] for k in rk], dtype=np.float32)
    a["rt_active"] = np.asarray([ut.root_tiles[k][1] for k in rk], dtype=bool)
    a["l2_origin"] = np.asarray([n.origin for n in ut.l2_nodes], dtype=np.int64).reshape(-1, 3)
    a["l2_child"] = np.packbits(np.asarray([n.child_mask.bits for n in ut.l2_nodes], dtype=bool).reshape(-1, L2_SIZE), axis=1)
    a["l2_active"] = np.packbits(np.asarray([n.active_mask.bits for n in ut.l2_nodes], dtype=bool).reshape(-1, L2_SIZE), axis=1)
    t = [(ni, k, v) for ni, n in enumerate(ut.l2_nodes) for k, v in sorted(n.tiles.items())]
    a["l2_tiles"] = np.asarray(t, dtype=np.float64).reshape(-1, 3)
    a["l1_origin"] = np.asarray(ut.l1_origins, dtype=np.int64).reshape(-1, 3)
    t = [(*o, k, v) for o, d in sorted(ut.l1_tiles.items()) for k, v in sorted(d.items())]
    a["l1_tiles"] = np.asarray(t, dtype=np.float64).reshape(-1, 5)
    nk, nb = _copy_leaf_bits(ut.leaf_negative_fill).arrays()
    order = np.lexsort((nk[:, 2], nk[:, 1], nk[:, 0])) if nk.shape[0] else np.zeros(0, np.int64)
    a["neg_origin"] = nk[order].reshape(-1, 3)
    a["neg_bits"] = np.packbits(nb[order].reshape(-1, LEAF_SIZE), axis=1)
    lay = c.layout
    a["layout"] = np.array([lay.size, lay.halo, lay.cluster_count], dtype=np.int64)
    a["sub_cells"] = np.asarray([[*s.cell, s.cluster_id] for s in lay.subdomains], dtype=np.int64).reshape(-1, 4)
    a["n_experts"] = np.array([len(c.experts)])
    for ei, e in enumerate(c.experts):
        p = f"e{ei}_"
        a[p + "hdr"] = np.array([e.id, *e.cell, e.cluster_id], dtype=np.int64)
        a[p + "norm"] = np.array([*e.norm_origin, e.norm_scale, e.value_scale], dtype=np.float64)
        for tag, net in e.nets():
            if net is None:
                continue
            q = p + tag + "_"
            pr = net.params
            a[q + "hdr"] = np.array([len(pr.layers), _ACT[pr.activation.kind], pr.activation.frequency,
                                     _HEAD[pr.head], net.ff.seed, net.ff.scale, net.ff.m,
                                     net.ff.amplitude, net.final_loss, net.epochs], dtype=np.float64)
            a[q + "seed"] = np.array([net.ff.seed], dtype=np.uint64)
            for li, (w, b) in enumerate(pr.layers):
                a[q + f"w{li}"] = np.asarray(w, dtype=np.float32)
                a[q + f"b{li}"] = np.asarray(b, dtype=np.float32)
        k1, c1 = _patch_records(1, e.patches.l1).arrays()
        k0, a0, v0 = _patch_records(0, e.patches.l0).arrays()
        a[p + "pl1"] = np.concatenate([k1, c1[:, None]], axis=1).astype(np.int64).reshape(-1, 4)
        a[p + "pl0"] = np.concatenate([k0, a0[:, None].astype(np.int64)], axis=1).reshape(-1, 4)
        a[p + "pl0v"] = np.asarray(v0, dtype=np.float64).copy()
    return {prefix + k: v for k, v in a.items()}


def container_from_arrays(a, prefix: str = "c_") -> NeuralGridContainer:
    g = lambda k: a[prefix + k]  # noqa: E731
    meta_a = g("meta")
    meta = GridMeta(GRID_CLASS_SDF if meta_a[0] == 0 else GRID_CLASS_FOG, float(meta_a[1]),
                    float(meta_a[2]), float(meta_a[3]), float(meta_a[4]))
    tree = UpperTree()
    for o, v, act in zip(g("rt_origin"), g("rt_value"), g("rt_active")):
        tree.root_tiles[tuple(int(x) for x in o)] = (float(v), bool(act))
    l2c = np.unpackbits(g("l2_child"), axis=1, count=L2_SIZE).astype(bool)
    l2a = np.unpackbits(g("l2_active"), axis=1, count=L2_SIZE).astype(bool)
    for ni, o in enumerate(g("l2_origin")):
        tree.l2_nodes.append(L2NodeRecord(tuple(int(x) for x in o), Mask(l2c[ni]), Mask(l2a[ni]), {}))
    for ni, k, v in g("l2_tiles"):
        tree.l2_nodes[int(ni)].tiles[int(k)] = float(v)
    tree.l1_origins = [tuple(int(x) for x in o) for o in g("l1_origin")]
    for x, y, z, k, v in g("l1_tiles"):
        tree.l1_tiles.setdefault((int(x), int(y), int(z)), {})[int(k)] = float(v)
    nb = np.unpackbits(g("neg_bits"), axis=1, count=LEAF_SIZE).astype(bool)
    tree.leaf_negative_fill = LeafBitsMap.from_arrays(np.asarray(g("neg_origin"), np.int64).reshape(-1, 3),
                                                      nb.reshape(-1, LEAF_SIZE))
    size, halo, ccount = (int(v) for v in g("layout"))
    layout = SubdomainLayout(size=size, halo=halo, cluster_count=ccount)
    for sid, row in enumerate(g("sub_cells")):
        cell = tuple(int(v) for v in row[:3])
        layout.subdomains.append(Subdomain(sid, cell, size, int(row[3]), halo))
        layout.cell_to_id[cell] = sid
    experts = []
    for ei in range(int(g("n_experts")[0])):
        p = f"e{ei}_"
        hdr = g(p + "hdr")
        norm = g(p + "norm")
        ex = EncodedSubdomain(int(hdr[0]), tuple(int(v) for v in hdr[1:4]), int(hdr[4]),
                              norm[:3].copy(), float(norm[3]), float(norm[4]))
        for tag, attr in (("l1", "l1_classifier"), ("tile", "tile_regressor"),
                          ("l0", "l0_classifier"), ("voxel", "voxel_regressor")):
            q = p + tag + "_"
            if prefix + q + "hdr" not in a:
                continue
            h = g(q + "hdr")
            nl = int(h[0])
            layers = [(g(q + f"w{li}").copy(), g(q + f"b{li}").copy()) for li in range(nl)]
            seed = int(g(q + "seed")[0])
            ff = FourierFeatures(int(h[6]), float(h[5]), seed, float(h[7]))
            params = MlpParams(layers, Activation(_INV_ACT[int(h[1])], float(h[2])), _INV_HEAD[int(h[3])])
            setattr(ex, attr, NetRecord(params, ff, float(h[8]), int(h[9])))
        ex.patches = PatchList()
        r1, r0 = np.asarray(g(p + "pl1"), np.int64).reshape(-1, 4), np.asarray(g(p + "pl0"), np.int64).reshape(-1, 4)
        ex.patches.l1.extend_arrays(r1[:, :3], r1[:, 3])
        ex.patches.l0.extend_arrays(r0[:, :3], r0[:, 3] != 0, np.asarray(g(p + "pl0v"), np.float64).reshape(-1))
        experts.append(ex)
    return NeuralGridContainer(meta, tree, layout, experts, None, 32)


def grid_to_arrays(grid: DenseLeafGrid, prefix: str = "g_") -> Dict[str, np.ndarray]:
    a = {
        "meta": np.array([0 if grid.grid_class == GRID_CLASS_SDF else 1, grid.background,
                          grid.voxel_size, grid.half_width], dtype=np.float64),
        "rt_origin": np.asarray(sorted(grid.root_tiles), dtype=np.int64).reshape(-1, 3),
        "rt_val": np.asarray([grid.root_tiles[k][0] for k in sorted(grid.root_tiles)], dtype=np.float32),
        "rt_act": np.asarray([grid.root_tiles[k][1] for k in sorted(grid.root_tiles)], dtype=bool),
        "l2_origins": grid.l2_origins, "l2_child": np.packbits(grid.l2_child, axis=1),
        "l2_active": np.packbits(grid.l2_active, axis=1), "l2_tiles": grid.l2_tiles,
        "l1_origins": grid.l1_origins, "l1_child": np.packbits(grid.l1_child, axis=1),
        "l1_active": np.packbits(grid.l1_active, axis=1), "l1_tiles": grid.l1_tiles,
        "leaf_origins": grid.leaf_origins, "leaf_active": np.packbits(grid.leaf_active, axis=1),
        "leaf_values": grid.leaf_values,
    }
    return {prefix + k: v for k, v in a.items()}


def grid_from_arrays(a, prefix: str = "g_") -> DenseLeafGrid:
    g = lambda k: a[prefix + k]  # noqa: E731
    meta = g("meta")
    rt = {tuple(int(x) for x in o): (float(v), bool(act))
          for o, v, act in zip(g("rt_origin"), g("rt_val"), g("rt_act"))}
    return DenseLeafGrid(
        background=float(meta[1]), grid_class=GRID_CLASS_SDF if meta[0] == 0 else GRID_CLASS_FOG,
        voxel_size=float(meta[2]), half_width=float(meta[3]), root_tiles=rt,
        l2_origins=g("l2_origins").astype(np.int64),
        l2_child=np.unpackbits(g("l2_child"), axis=1, count=L2_SIZE).astype(bool),
        l2_active=np.unpackbits(g("l2_active"), axis=1, count=L2_SIZE).astype(bool),
        l2_tiles=g("l2_tiles").astype(np.float32),
        l1_origins=g("l1_origins").astype(np.int64),
        l1_child=np.unpackbits(g("l1_child"), axis=1, count=L1_SIZE).astype(bool),
        l1_active=np.unpackbits(g("l1_active"), axis=1, count=L1_SIZE).astype(bool),
        l1_tiles=g("l1_tiles").astype(np.float32),
        leaf_origins=g("leaf_origins").astype(np.int64),
        leaf_active=np.unpackbits(g("leaf_active"), axis=1, count=LEAF_SIZE).astype(bool),
        leaf_values=g("leaf_values").astype(np.float32),
    )


def _copy_patches(pl) -> PatchList:
    """A PatchList of PatchRecords from any patch container (reference lists of tuples included)."""
    out = PatchList()
    for level, src, dst in ((1, pl.l1, out.l1), (0, pl.l0, out.l0)):
        cols = _patch_records(level, src).arrays()
        dst.extend_arrays(*[c.copy() for c in cols])
    return out


def _copy_leaf_bits(m) -> LeafBitsMap:
    """A LeafBitsMap copy of any {origin: bits} mapping (reference dicts included)."""
    if isinstance(m, LeafBitsMap):
        k, b = m.arrays()
        return LeafBitsMap.from_arrays(k, b)
    out = LeafBitsMap()
    for k, v in m.items():
        out[k] = np.asarray(v, dtype=bool).reshape(-1).copy()
    out.arrays()
    return out
