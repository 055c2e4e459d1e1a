"""CPU tests of the host-side logic and the C-ABI boundary (no GPU needed)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_2208_04448_b200 import _lib
from paper_2208_04448_b200.model import grid_from_arrays
from paper_2208_04448_b200.tree import tree_arrays

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_symbols():
    text = open(os.path.join(ROOT, "include", "nvdb_b200.h")).read()
    return sorted(set(re.findall(r"NVDB_API [^;(]*?\b(nvdb_\w+)\s*\(", text)))


def test_header_matches_binding_list():
    assert _header_symbols() == sorted(_lib.EXPORTED)


def test_library_exports_every_header_symbol():
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("library not built (run __graft_entry__.build())")
    lib = C.CDLL(_lib.LIB_PATH)
    for name in _header_symbols():
        assert hasattr(lib, name), name
    L = _lib.lib()
    assert L.nvdb_version() >= 1


def _emulate_lookup(arr, background, coords):
    """numpy replay of csrc/lookup.cu's traversal on the packed tree arrays."""
    out_v = np.full(len(coords), background, np.float32)
    out_a = np.zeros(len(coords), np.uint8)
    out_k = np.zeros(len(coords), np.uint8)
    keys = {tuple(k): i for i, k in enumerate(arr["root_keys"])}

    def bit(words, node, wpn, idx):
        w = int(words[node, idx >> 6])
        return (w >> (idx & 63)) & 1, w

    def rank(words, node, idx, base):
        w = int(words[node, idx >> 6])
        below = sum(bin(int(words[node, j])).count("1") for j in range(idx >> 6))
        return int(base[node]) + below + bin(w & ((1 << (idx & 63)) - 1)).count("1")

    for i, (x, y, z) in enumerate(coords):
        r = keys.get((x & ~4095, y & ~4095, z & ~4095))
        if r is None:
            continue
        n2 = arr["root_l2"][r]
        if n2 < 0:
            out_v[i], out_a[i], out_k[i] = arr["root_tile_value"][r], arr["root_tile_active"][r], 1
            continue
        i2 = (((x & 4095) >> 7) << 10) | (((y & 4095) >> 7) << 5) | ((z & 4095) >> 7)
        c2, _ = bit(arr["l2_child"], n2, 512, i2)
        if not c2:
            out_v[i] = arr["l2_tiles"][n2, i2]
            out_a[i] = bit(arr["l2_active"], n2, 512, i2)[0]
            out_k[i] = 1
            continue
        n1 = rank(arr["l2_child"], n2, i2, arr["l2_child_base"])
        i1 = (((x & 127) >> 3) << 8) | (((y & 127) >> 3) << 4) | ((z & 127) >> 3)
        c1, _ = bit(arr["l1_child"], n1, 64, i1)
        if not c1:
            out_v[i] = arr["l1_tiles"][n1, i1]
            out_a[i] = bit(arr["l1_active"], n1, 64, i1)[0]
            out_k[i] = 1
            continue
        lf = rank(arr["l1_child"], n1, i1, arr["l1_child_base"])
        i0 = ((x & 7) << 6) | ((y & 7) << 3) | (z & 7)
        out_v[i] = arr["leaf_values"][lf, i0]
        out_a[i] = bit(arr["leaf_active"], lf, 8, i0)[0]
        out_k[i] = 2
    return out_v, out_a, out_k


def test_packed_tree_layout_resolves_reference_lookups(golden):
    """The packed tree the CUDA lookup walks reproduces get_values exactly."""
    z = golden("lookup_small")
    g = grid_from_arrays(z)
    arr = tree_arrays(g)
    sel = np.arange(0, len(z["coords"]), 7)
    v, a, k = _emulate_lookup(arr, g.background, [tuple(int(t) for t in c) for c in z["coords"][sel]])
    np.testing.assert_array_equal(v.view(np.uint32), z["values"][sel].view(np.uint32))
    np.testing.assert_array_equal(a.astype(bool), z["active"][sel])
    np.testing.assert_array_equal(k, z["kind"][sel])
