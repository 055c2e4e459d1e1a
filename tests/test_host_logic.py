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


def test_patch_arrays_later_expert_overrides_like_a_dict():
    """decoder.py:84-92: patch maps are dicts filled expert by expert."""
    from paper_2208_04448_b200.decoder import _patch_arrays
    rng = np.random.default_rng(3)
    lists = []
    for e in range(3):
        keys = [tuple(int(v) for v in rng.integers(-64, 64, 3)) for _ in range(200)]
        lists.append([(k, bool(rng.integers(0, 2)), float(rng.normal())) for k in keys])
    ref = {}
    for lst in lists:
        for k, a, v in lst:
            ref[k] = (a, v)
    keys, act, val = _patch_arrays(lists, 2)
    got = {tuple(int(x) for x in k): (bool(a), float(v)) for k, a, v in zip(keys, act, val)}
    assert got == ref and keys.shape[0] == len(ref)
    k1, c1 = _patch_arrays([[((0, 8, 16), 2)], [], [((0, 8, 16), 1), ((8, 8, 8), 0)]], 1)
    assert {tuple(int(x) for x in k): int(c) for k, c in zip(k1, c1)} == {(0, 8, 16): 1, (8, 8, 8): 0}
    k0, c0 = _patch_arrays([[], []], 1)
    assert k0.shape == (0, 3) and c0.shape == (0,)
    # the same through array-backed records (model.PatchRecords), mixed with plain lists
    from paper_2208_04448_b200.model import PatchRecords
    recs = [PatchRecords(0, lists[0]), lists[1], PatchRecords(0)]
    recs[2].extend_arrays(np.array([k for k, _, _ in lists[2]]), np.array([a for _, a, _ in lists[2]]),
                          np.array([v for _, _, v in lists[2]]))
    keys2, act2, val2 = _patch_arrays(recs, 2)
    np.testing.assert_array_equal(keys2, keys)
    np.testing.assert_array_equal(act2, act)
    np.testing.assert_array_equal(val2, val)


def test_patch_records_behave_like_the_reference_lists():
    """container.py:100-117 / 345-351 / 455-460: PatchList.l1 / .l0 are lists of
    (origin, cls) / (coord, active, value) that the encoder appends to and the
    writer iterates."""
    import pickle
    from paper_2208_04448_b200.model import (PatchList, container_from_arrays, container_to_arrays)
    ref0 = [((70, 127, 247), True, 2.963477849960327), ((-8, 0, 5), False, 0.0), ((1, 2, 3), True, -0.25)]
    ref1 = [((0, 0, 128), 2), ((-128, 8, 16), 0)]
    pl = PatchList()
    for r in ref0:
        pl.l0.append(r)
    pl.l1.extend_arrays(np.array([k for k, _ in ref1]), np.array([c for _, c in ref1]))
    assert list(pl.l0) == ref0 and pl.l0 == ref0 and pl.l1 == ref1 and len(pl) == 5
    assert pl.l0[1] == ref0[1] and pl.l0[-1] == ref0[-1] and pl.l1[0:1] == ref1[0:1]
    assert [type(x) for x in pl.l0[0]] == [tuple, bool, float] and type(pl.l0[0][0][0]) is int
    with pytest.raises(IndexError):
        pl.l1[2]
    assert pickle.loads(pickle.dumps(pl)) == pl
    assert PatchList(l1=ref1, l0=ref0) == pl
    with pytest.raises(ValueError):
        pl.l0.extend_arrays(np.zeros((2, 3)), np.zeros(2, bool), np.zeros(3))
    # container arrays round trip keeps the records
    from conftest import load_golden
    c = container_from_arrays(load_golden("decode_multi"))
    assert sum(len(e.patches) for e in c.experts) > 0
    c2 = container_from_arrays(container_to_arrays(c))
    for a, b in zip(c.experts, c2.experts):
        assert a.patches == b.patches


def test_node_index_matches_dict_lookup():
    """DeviceModel._node_index (dense code + searchsorted) == {origin: index}."""
    from paper_2208_04448_b200.decoder import DeviceModel
    rng = np.random.default_rng(4)
    origins = np.unique(rng.integers(-20, 20, size=(300, 3)) * 128, axis=0).astype(np.int64)
    m = DeviceModel.__new__(DeviceModel)
    m.origins, m.n1 = origins, origins.shape[0]
    lut = {tuple(o): i for i, o in enumerate(origins.tolist())}
    keys = np.concatenate([origins[rng.permutation(len(origins))[:150]],
                           rng.integers(-30, 30, size=(300, 3)) * 128,
                           rng.integers(-3000, 3000, size=(50, 3))]).astype(np.int64)
    got = m._node_index(keys)
    ref = np.array([lut.get(tuple(k), -1) for k in keys.tolist()])
    np.testing.assert_array_equal(got, ref)
    assert (m._node_index(np.zeros((0, 3), np.int64)) == 0).all()
    # a bounding box too large for the direct table (binary-search path)
    far = origins.copy()
    far[::2, 0] += np.int64(1 << 36)
    m2 = DeviceModel.__new__(DeviceModel)
    m2.origins, m2.n1 = far, far.shape[0]
    lut2 = {tuple(o): i for i, o in enumerate(far.tolist())}
    keys2 = np.concatenate([far[rng.permutation(len(far))[:150]], keys]).astype(np.int64)
    np.testing.assert_array_equal(m2._node_index(keys2), np.array([lut2.get(tuple(k), -1) for k in keys2.tolist()]))
    assert m2._nidx[4] is None and m._nidx[4] is not None


def test_node_arrays_of_no_leaves():
    from paper_2208_04448_b200.procgen import _nodes_from_leaves
    l1o, l1c, l1a, l1t, l2o, l2c, l2a, l2t = _nodes_from_leaves(np.zeros((0, 3), np.int64), np.float32(0))
    assert l1o.shape == (0, 3) and l2o.shape == (0, 3) and l1c.shape[0] == 0 and l2c.shape[0] == 0


def test_bench_reads_committed_traffic():
    import bench
    t = bench.load_traffic()
    assert t is not None and t["bytes_per_launch"] > 0 and os.path.exists(os.path.join(bench.ROOT, t["source"]))


def test_leaf_bits_map_behaves_like_the_reference_dict():
    """UpperTree.leaf_negative_fill (encoder.py:519-526) is a {leaf origin: (512,) bool} dict."""
    import pickle
    from paper_2208_04448_b200.model import LeafBitsMap
    rng = np.random.default_rng(0)
    d, m = {}, LeafBitsMap()
    for _ in range(50):
        k = tuple(int(v) for v in rng.integers(-100, 100, 3) * 8)
        b = rng.random(512) < 0.3
        d[k] = b
        m[k] = b
    m2 = LeafBitsMap.from_arrays(*m.arrays())
    for k in list(d)[:10]:
        b = rng.random(512) < 0.5
        d[k] = b
        m2[k] = b
    d[(8, 8, 8)] = np.ones(512, bool)
    m2[(8, 8, 8)] = d[(8, 8, 8)]
    k3 = list(d)[3]
    del d[k3]
    del m2[k3]
    assert list(d) == list(m2) and len(d) == len(m2) and all((d[k] == m2[k]).all() for k in d)
    assert (8, 8, 8) in m2 and (1, 2, 3) not in m2
    with pytest.raises(KeyError):
        m2[(1, 2, 3)]
    m3 = pickle.loads(pickle.dumps(m2))
    assert list(m3) == list(m2) and all((m3[k] == m2[k]).all() for k in d)
    keys, bits = m3.arrays()
    assert keys.shape == (len(d), 3) and bits.shape == (len(d), 512) and bits.dtype == bool
    with pytest.raises(ValueError):
        LeafBitsMap.from_arrays(np.zeros((2, 3)), np.zeros((2, 512), bool))  # duplicate origins


def test_training_input_errors_match_reference():
    """neural.py:282-283, 295-296, 309-310: NaN inputs, CE labels outside the
    head and non-binary BCE targets raise ValueError, before any device work."""
    import sys
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from helpers import tiny_cfg
    from paper_2208_04448_b200.encoder import net_spec, train_network
    cfg = tiny_cfg()
    x = np.zeros((10, 3), np.float32)
    xn = x.copy()
    xn[3, 1] = np.nan
    for xx, yy, tag, msg in ((xn, np.zeros(10, np.float32), "voxel", "NaN"),
                             (x, np.full(10, 5), "l1", "label"),
                             (x, np.full(10, -1), "l1", "label"),
                             (x, np.full(10, 0.5, np.float32), "l0", "binary"),
                             (x, np.array([0, 1, np.nan, 0, 1, 0, 0, 1, 1, 0], np.float32), "voxel", "NaN")):
        with pytest.raises(ValueError, match=msg):
            train_network(xx, yy, net_spec(tag, cfg), cfg, 0, cfg.lr)


def test_committed_bench_line_keeps_the_contract():
    """profiles/r01/bench_c2_final.json (a real bench.py line) carries every key
    the driver and the judge read."""
    import json
    d = json.load(open(os.path.join(ROOT, "profiles", "r01", "bench_c2_final.json")))
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e",
              "gpu_launches", "clocks"):
        assert k in d, k
    assert d["config"]["workload"] and d["warmup"] >= 3 and d["gpu_launches"] > 0
    r = d["roofline"]
    assert r["bound"] in ("hbm", "tensor") and r["peak"] > 0 and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    assert "traffic" in r and r["co_bound"]["bound"] == "mufu"
    cb = d["cpu_baseline"]
    assert cb["kind"] in ("reference", "port") and cb["cores"] >= 1 and cb["value"] > 0 and cb["sample"]
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    c = d["clocks"]
    assert c["sm_mhz"] > 0 and not set(c["reasons"]) & {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}


def test_host_training_setup_matches_reference(golden):
    """init_mlp (neural.py:168-185), decompose (partition.py:74-120),
    _expert_norm and _gather_expert_data (encoder.py:181-235) against the
    reference's own outputs (tests/golden/make_golden_host.py): an 8-expert
    straddling sphere, a torus around a lattice line (4 experts) and a FOG
    grid; bit-exact."""
    from paper_2208_04448_b200.encoder import decompose, expert_norm, gather_expert_data, init_mlp, value_scale_of
    from paper_2208_04448_b200.model import Activation, grid_from_arrays
    z = golden("host_setup")
    cases = [(384, [96, 96, 96], 1, "sine", 3.0, "linear", 11), (96, [48, 48, 48], 3, "sine", 3.0, "logits", 12),
             (512, [256, 256, 256], 1, "sine", 1.5, "binary", 13), (40, [24, 24], 1, "relu", 1.0, "linear", 14),
             (64, [100, 60], 3, "tanh", 1.0, "logits", 15)]
    for i, (ind, hid, od, act, fr, head, seed) in enumerate(cases):
        p = init_mlp(ind, hid, od, Activation(act, fr), head, seed)
        for li, (w, b) in enumerate(p.layers):
            np.testing.assert_array_equal(w, z[f"init{i}_w{li}"])
            np.testing.assert_array_equal(b, z[f"init{i}_b{li}"])
            assert w.dtype == z[f"init{i}_w{li}"].dtype
    for name in ("straddle", "torus", "fog"):
        g = grid_from_arrays(z, f"{name}_g_")
        layout = decompose(g, 512)
        np.testing.assert_array_equal(np.array([s.cell for s in layout.subdomains]), z[f"{name}_cells"])
        np.testing.assert_array_equal(np.array([s.cluster_id for s in layout.subdomains]), z[f"{name}_clusters"])
        scale = value_scale_of(g)
        for s in layout.subdomains:
            q = f"{name}_e{s.id}_"
            no, ns = expert_norm(s, g)
            np.testing.assert_array_equal(np.array([*no, ns]), z[q + "norm"])
            d = gather_expert_data(g, s, scale)
            for k in ("l1_inputs", "l1_labels", "l0_inputs", "l0_labels", "vox_inputs", "vox_targets"):
                v = getattr(d, k)
                ref = z[q + k]
                if v is None:
                    assert ref.size == 0, (name, s.id, k)
                    continue
                np.testing.assert_array_equal(v, ref, err_msg=f"{name} expert {s.id} {k}")
                assert v.dtype == ref.dtype, (k, v.dtype, ref.dtype)
