"""Pin the CPU oracle against vectors produced by the reference itself.

The fixtures were generated with OPENBLAS_NUM_THREADS=1; sgemm blocking
changes the summation order with the thread count, so float comparisons use
a 1e-5 tolerance (the reference's own fused-vs-canonical bar,
test_neural.py:244-270) while integer/index/mask results are exact.
"""
import numpy as np
import pytest

import oracle as O
from helpers import ACTS, HEADS, LOSSES, net_from_fixture, tiny_cfg
from paper_2208_04448_b200.model import (Activation, FourierFeatures, MlpParams,
                                         container_from_arrays, grid_from_arrays)


def test_forward_block_matches_reference(golden):
    z = golden("nets")
    for ci in range(int(z["ncases"][0])):
        q = f"n{ci}_"
        params, ff = net_from_fixture(z, q)
        y = O.forward_block(params, ff, z[q + "pts"])
        np.testing.assert_allclose(y, z[q + "out"], rtol=1e-5, atol=1e-5)


def test_train_step_matches_reference(golden):
    z = golden("steps")
    for ci in range(int(z["ncases"][0])):
        q = f"s{ci}_"
        cfg = z[q + "cfg"]
        kind, freq, m, od = ACTS[int(cfg[0])], float(cfg[1]), int(cfg[2]), int(cfg[3])
        hidden = list(z[q + "hidden"])
        ff = FourierFeatures(m, 5.0, int(cfg[5]))
        layers = O.init_layers(2 * m, hidden, od, kind, freq, int(cfg[6]))
        st = O.TrainState(layers, kind, freq, ff)
        losses = []
        for step in range(6):
            lr = np.float32(O.lr_at(1e-3, 0.975, 100.0, step))
            losses.append(O.train_step(st, z[q + "xb"], z[q + "yb"], LOSSES[int(cfg[7])], lr))
        np.testing.assert_allclose(losses, z[q + "losses"], rtol=1e-5)
        for li, (w, b) in enumerate(st.layers_interleaved()):
            np.testing.assert_allclose(w, z[q + f"w{li}"], atol=1e-5)
            np.testing.assert_allclose(b, z[q + f"b{li}"], atol=1e-5)


def test_sampler_bit_exact(golden):
    z = golden("sampler")
    for ci in range(int(z["ncases"][0])):
        n, b, iv, seed = (int(v) for v in z[f"c{ci}_cfg"])
        s = O.Sampler(n, b, iv, seed)
        for ep in z[f"c{ci}_epochs"]:
            np.testing.assert_array_equal(s.indices(int(ep)), z[f"c{ci}_e{int(ep)}"])
    for parts, val in zip(z["seed_parts"], z["seed_vals"]):
        assert O.stable_seed(*[int(p) for p in parts if p >= 0]) == int(val)


def test_lookup_bit_exact(golden):
    z = golden("lookup_small")
    g = grid_from_arrays(z)
    v, a, k = O.lookup(g, z["coords"])
    np.testing.assert_array_equal(v.view(np.uint32), z["values"].view(np.uint32))
    np.testing.assert_array_equal(a, z["active"])
    np.testing.assert_array_equal(k, z["kind"])


def test_coord_keys_known_answers():
    root, i2, i1, i0 = O.coord_keys(np.array([[-1, -1, -1], [4096, 0, 0], [0, 0, 0]]))
    assert tuple(root[0]) == (-4096, -4096, -4096)
    assert (i2[0], i1[0], i0[0]) == (32767, 4095, 511)
    assert tuple(root[1]) == (4096, 0, 0) and (i2[1], i1[1], i0[1]) == (0, 0, 0)


@pytest.mark.parametrize("name", ["decode_small", "decode_multi"])
def test_decode_matches_reference(golden, name):
    z = golden(name)
    c = container_from_arrays(z)
    d = grid_from_arrays(z, "d_")
    r = O.decode(c)
    # leaves keyed by origin (node order differs only across level-2 nodes)
    mine = {tuple(o): i for i, o in enumerate(r.leaf_origins)}
    assert len(mine) == d.leaf_origins.shape[0]
    idx = np.array([mine[tuple(o)] for o in d.leaf_origins])
    np.testing.assert_array_equal(r.leaf_active[idx], d.leaf_active)
    np.testing.assert_allclose(r.leaf_values[idx], d.leaf_values, atol=1e-6)
    assert r.regressor_evaluations == int(z["evals"][0])


@pytest.mark.parametrize("name", ["decode_small", "decode_multi"])
def test_blend_and_assign_match_reference(golden, name):
    z = golden(name)
    c = container_from_arrays(z)
    cen = z["cen"]
    for tag, pk, ck in (("l1", "p1", "c1"), ("l0", "p0", "c0"), ("voxel", "pv", "cv")):
        p, cov = O.blended(c.layout, c.experts, cen, tag)
        np.testing.assert_array_equal(cov, z[ck])
        np.testing.assert_allclose(p.reshape(z[pk].shape), z[pk], atol=1e-6)
    asg = O.assign(c.layout, cen)
    rows = np.concatenate([np.stack([np.full(len(r), s), r], 1) for s, (r, w) in sorted(asg.items())])
    w = np.concatenate([w for s, (r, w) in sorted(asg.items())])
    np.testing.assert_array_equal(rows, z["asg_rows"])
    np.testing.assert_array_equal(w, z["asg_w"])


@pytest.mark.parametrize("name", ["decode_small", "decode_multi"])
def test_hybrid_query_matches_reference(golden, name):
    z = golden(name)
    c = container_from_arrays(z)
    topo = O.decode(c, materialize_values=False)
    v, a, ev = O.hybrid_query(c, topo, z["q"])
    np.testing.assert_array_equal(a, z["qa"])
    np.testing.assert_allclose(v, z["qv"], atol=1e-6)
    assert ev == int(z["evals"][1])


def test_train_network_matches_reference(golden):
    z = golden("train_small")
    cf = z["cfg"]
    cfg = tiny_cfg(l1_net=(int(cf[0]), int(cf[1])), l0_net=(int(cf[2]), int(cf[3])),
                   voxel_net=(int(cf[4]), int(cf[5])), ffm_size=int(cf[6]), max_epochs=int(cf[7]),
                   batch_size=int(cf[8]), seed=int(cf[9]), frequency=float(cf[10]),
                   ffm_scale=float(cf[11]), lr=float(cf[12]))
    for tag in ("l1", "l0", "voxel"):
        spec = O.net_spec(tag, cfg)
        layers, ff, loss, ep = O.train_network(z[tag + "_x"], z[tag + "_y"], spec, cfg, 0, cfg.lr)
        assert ep == int(z[tag + "_loss"][1])
        np.testing.assert_allclose(loss, z[tag + "_loss"][0], rtol=1e-5)
        for li, (w, b) in enumerate(layers):
            np.testing.assert_allclose(w, z[tag + f"_w{li}"], atol=1e-5)
            np.testing.assert_allclose(b, z[tag + f"_b{li}"], atol=1e-5)
