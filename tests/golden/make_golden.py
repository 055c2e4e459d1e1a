"""Generate golden fixtures by running the reference package itself.

Run in the build container (the reference is not present on the GPU box):

    PYTHONPATH=/root/reference/pkg/src:/root/repo PYTHONDONTWRITEBYTECODE=1 \
    OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden.py [--c1 /tmp/gw/c1.nvdb]

Every fixture is a compressed ``.npz`` of inputs and the reference's outputs
for them.  ``tests/test_oracle_golden.py`` pins the oracle against these;
the GPU parity tests compare the CUDA path against the oracle and these.
The C1 fixture (sphere 128^3, ACCEPT_CONFIG, fp16 container) comes from an
encode that takes ~7 min on 8 cores; pass its serialized container with
``--c1`` (written by ``tests/golden/run_c1_encode.py``).
"""

from __future__ import annotations

import argparse
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from svcodec import neural as N  # noqa: E402
from svcodec.config import TrainConfig  # noqa: E402
from svcodec.container import deserialize_container  # noqa: E402
from svcodec.decoder import decode_full, decode_report, make_hybrid  # noqa: E402
from svcodec.encoder import Sampler, _net_spec, _stable_seed, encode, train_network, _flatten_grid, _gather_expert_data, _value_scale  # noqa: E402
from svcodec.inference import blended_l0_probs, blended_l1_probs, blended_values  # noqa: E402
from svcodec.partition import assign_points, decompose  # noqa: E402
from svcodec.procgen import SphereSpec, gen_sphere_sdf  # noqa: E402

from paper_2208_04448_b200.model import (DenseLeafGrid, container_to_arrays,  # noqa: E402
                                         grid_to_arrays)


def save(name, **arrays):
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **arrays)
    print(f"{name}: {os.path.getsize(path) / 1024:.1f} KiB")


def nets_fixture():
    rng = np.random.default_rng(7)
    out = {}
    cases = [("relu", 1.0, 8, [16, 16], 1, "linear"),
             ("tanh", 1.0, 12, [32, 32, 32], 3, "logits"),
             ("sine", 3.0, 16, [48, 48, 48], 3, "logits"),
             ("sine", 3.0, 32, [96, 96, 96], 1, "binary"),
             ("sine", 1.5, 20, [40, 24], 1, "linear")]
    for ci, (kind, freq, m, hidden, od, head) in enumerate(cases):
        act = N.Activation(kind, freq)
        ff = N.FourierFeatures(m, 5.0, 100 + ci)
        p = N.init_mlp(2 * m, hidden, od, act, head, 200 + ci)
        # non-zero head so outputs are informative
        w, b = p.layers[-1]
        w[...] = rng.uniform(-0.3, 0.3, size=w.shape).astype(np.float32)
        b[...] = rng.uniform(-0.1, 0.1, size=b.shape).astype(np.float32)
        for li, (wl, bl) in enumerate(p.layers[:-1]):
            bl[...] = rng.uniform(-0.2, 0.2, size=bl.shape).astype(np.float32)
        pts = rng.uniform(0.05, 0.95, size=(3000, 3)).astype(np.float32)
        y = N.forward_block(p, ff, pts)
        q = f"n{ci}_"
        out[q + "cfg"] = np.array([["relu", "tanh", "sine"].index(kind), freq, m, od,
                                   ["linear", "logits", "binary"].index(head), 100 + ci, 5.0])
        out[q + "hidden"] = np.array(hidden)
        for li, (wl, bl) in enumerate(p.layers):
            out[q + f"w{li}"] = wl
            out[q + f"b{li}"] = bl
        out[q + "pts"] = pts
        out[q + "out"] = y
    out["ncases"] = np.array([len(cases)])
    save("nets", **out)


def step_fixture():
    rng = np.random.default_rng(11)
    out = {}
    cases = [("sine", 3.0, "mse", 16, [32, 32, 32], 1, "linear"),
             ("sine", 3.0, "ce", 12, [24, 24, 24], 3, "logits"),
             ("sine", 3.0, "bce", 16, [32, 32, 32], 1, "binary"),
             ("relu", 1.0, "mse", 8, [16, 16], 1, "linear"),
             ("tanh", 1.0, "bce", 8, [16, 16], 1, "binary")]
    for ci, (kind, freq, loss, m, hidden, od, head) in enumerate(cases):
        act = N.Activation(kind, freq)
        ff = N.FourierFeatures(m, 5.0, 300 + ci)
        p = N.init_mlp(2 * m, hidden, od, act, head, 400 + ci)
        n = 1024
        xb = rng.uniform(0.0, 1.0, size=(n, 3)).astype(np.float32)
        if loss == "mse":
            yb = rng.uniform(-1, 1, size=n).astype(np.float32)
        elif loss == "ce":
            yb = rng.integers(0, 3, size=n).astype(np.int64)
        else:
            yb = (rng.uniform(size=n) < 0.4).astype(np.float32)
        net = N.FusedNet(p, ff)
        ws = N.TrainWorkspace()
        losses = []
        for step in range(6):
            lr = np.float32(N.lr_at(N.LrSchedule(1e-3, 0.975, 100.0), step))
            losses.append(N.fused_step(net, xb, yb, loss, lr, ws))
        net.commit()
        q = f"s{ci}_"
        out[q + "cfg"] = np.array([["relu", "tanh", "sine"].index(kind), freq, m, od,
                                   ["linear", "logits", "binary"].index(head), 300 + ci, 400 + ci,
                                   ["mse", "ce", "bce"].index(loss)])
        out[q + "hidden"] = np.array(hidden)
        out[q + "xb"] = xb
        out[q + "yb"] = yb
        out[q + "losses"] = np.array(losses)
        for li, (wl, bl) in enumerate(p.layers):
            out[q + f"w{li}"] = wl
            out[q + f"b{li}"] = bl
    out["ncases"] = np.array([len(cases)])
    save("steps", **out)


def sampler_fixture():
    out = {}
    cases = [(1000, 64, 1, 12345, [0, 1, 7]), (281936, 65536, 1, 3141592653, [0, 5]),
             (70000, 4096, 3, 99, [0, 1, 2, 3, 8]), (5, 17, 1, 1, [0]),
             (2 ** 31 + 11, 4096, 1, 77, [3])]
    for ci, (n, b, iv, seed, epochs) in enumerate(cases):
        s = Sampler(n, b, iv, seed)
        for ep in epochs:
            out[f"c{ci}_e{ep}"] = s.indices(ep).astype(np.int64)
        out[f"c{ci}_cfg"] = np.array([n, b, iv, seed], dtype=np.uint64)
        out[f"c{ci}_epochs"] = np.array(epochs)
    out["ncases"] = np.array([len(cases)])
    seeds = [(4242, 0, 2, 0), (4242, 0, 3, 2), (11, 1, 0, 1), (9000 + 3,), (1, 2, 3, 4)]
    out["seed_parts"] = np.array([list(s) + [-1] * (4 - len(s)) for s in seeds])
    out["seed_vals"] = np.array([_stable_seed(*s) for s in seeds], dtype=np.uint64)
    save("sampler", **out)


def small_sphere():
    return gen_sphere_sdf(SphereSpec(center=(20, 20, 20), radius=12.0, voxel_size=1.0,
                                     half_width=3.0))


def lookup_fixture(g, name):
    rng = np.random.default_rng(5)
    flat = DenseLeafGrid.from_svcodec(g)
    lo = flat.leaf_origins.min(axis=0) - 20
    hi = flat.leaf_origins.max(axis=0) + 28
    coords = rng.integers(lo, hi, size=(20000, 3))
    # plus exact active voxels, far negatives and the (-1,-1,-1) corner
    ac, _ = flat.active_voxels()
    extra = np.concatenate([ac[rng.integers(0, len(ac), 2000)],
                            rng.integers(-(2 ** 30) + 1, 2 ** 30 - 1, size=(500, 3)),
                            np.array([[-1, -1, -1], [0, 0, 0], [4095, 4095, 4095], [4096, 0, 0]])])
    coords = np.concatenate([coords, extra]).astype(np.int64)
    v, a, k = g.get_values(coords, with_kind=True)
    save(name, coords=coords, values=v, active=a, kind=k, **grid_to_arrays(flat))


def decode_fixture(g, cfg, name, nquery=20000):
    c = encode(g, cfg)
    d = decode_full(c)
    rep = decode_report(c)
    flat = DenseLeafGrid.from_svcodec(d)
    h = make_hybrid(c)
    rng = np.random.default_rng(3)
    lo = flat.leaf_origins.min(axis=0) - 10
    hi = flat.leaf_origins.max(axis=0) + 18
    q = rng.integers(lo, hi, size=(nquery, 3))
    ac, _ = flat.active_voxels()
    q = np.concatenate([q, ac[rng.integers(0, len(ac), 3000)]]).astype(np.int64)
    qv, qa = h.query(q)
    # raw blended evaluators on the decode's own centers
    cen = q[:4000].astype(np.float64) + 0.5
    p1, c1 = blended_l1_probs(c.layout, c.experts, cen)
    p0, c0 = blended_l0_probs(c.layout, c.experts, cen)
    pv, cv = blended_values(c.layout, c.experts, cen, "voxel")
    asg = assign_points(c.layout, cen)
    asg_rows = np.concatenate([np.stack([np.full(len(r), sid), r], 1) for sid, (r, w) in sorted(asg.items())]) if asg else np.zeros((0, 2))
    asg_w = np.concatenate([w for sid, (r, w) in sorted(asg.items())]) if asg else np.zeros(0)
    save(name, q=q, qv=qv, qa=qa, evals=np.array([rep["regressor_evaluations"], h.regressor_evaluations]),
         cen=cen, p1=p1, c1=c1, p0=p0, c0=c0, pv=pv, cv=cv, asg_rows=asg_rows, asg_w=asg_w,
         **container_to_arrays(c), **grid_to_arrays(flat, "d_"),
         **grid_to_arrays(DenseLeafGrid.from_svcodec(g), "g_"))
    return c


def train_fixture(g, cfg):
    """train_network on real expert data for l1/l0/voxel, few epochs."""
    layout = decompose(g, cfg.subdomain_size)
    arrays = _flatten_grid(g)
    data = _gather_expert_data(g, layout.subdomains[0], arrays, _value_scale(g))
    out = {"norm": np.array([*data.norm_origin, data.norm_scale])}
    for tag, x, y in (("l1", data.l1_inputs, data.l1_labels), ("l0", data.l0_inputs, data.l0_labels),
                      ("voxel", data.vox_inputs, data.vox_targets)):
        rec = train_network(x, y, _net_spec(tag, cfg), cfg, 0, cfg.lr)
        out[tag + "_x"] = x
        out[tag + "_y"] = y
        out[tag + "_loss"] = np.array([rec.final_loss, rec.epochs])
        for li, (w, b) in enumerate(rec.params.layers):
            out[tag + f"_w{li}"] = w
            out[tag + f"_b{li}"] = b
    out["cfg"] = np.array([cfg.l1_net[0], cfg.l1_net[1], cfg.l0_net[0], cfg.l0_net[1],
                           cfg.voxel_net[0], cfg.voxel_net[1], cfg.ffm_size, cfg.max_epochs,
                           cfg.batch_size, cfg.seed, cfg.frequency, cfg.ffm_scale, cfg.lr])
    save("train_small", **out)


def c1_fixture(path):
    blob = open(path, "rb").read()
    c = deserialize_container(blob)
    d = decode_full(c)
    flat = DenseLeafGrid.from_svcodec(d)
    rng = np.random.default_rng(17)
    q = rng.integers(0, 128, size=(20000, 3)).astype(np.int64)
    h = make_hybrid(c)
    qv, qa = h.query(q)
    li, vi = np.nonzero(flat.leaf_active)
    g = gen_sphere_sdf(SphereSpec(center=(63.5, 63.5, 63.5), radius=61.0, voxel_size=1.0, half_width=3.0))
    truth = DenseLeafGrid.from_svcodec(g)
    ti, tv = np.nonzero(truth.leaf_active)
    save("c1_sphere128", q=q, qv=qv, qa=qa, evals=np.array([decode_report(c)["regressor_evaluations"]]),
         truth_leaf_origins=truth.leaf_origins, truth_active=np.packbits(truth.leaf_active, axis=1),
         truth_values=truth.leaf_values[ti, tv],
         leaf_origins=flat.leaf_origins, leaf_active=np.packbits(flat.leaf_active, axis=1),
         active_values=flat.leaf_values[li, vi], l1_child=np.packbits(flat.l1_child, axis=1),
         l1_active=np.packbits(flat.l1_active, axis=1), **container_to_arrays(c))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--c1", default=None)
    ap.add_argument("--only", default=None)
    args = ap.parse_args()
    only = set(args.only.split(",")) if args.only else None

    def want(k):
        return only is None or k in only

    if want("nets"):
        nets_fixture()
    if want("steps"):
        step_fixture()
    if want("sampler"):
        sampler_fixture()
    g = small_sphere()
    tiny = TrainConfig(l1_net=(2, 8), l0_net=(2, 16), voxel_net=(2, 16), tile_net=None,
                       ffm_size=16, ffm_scale=5.0, max_epochs=40, batch_size=4096, seed=11)
    if want("lookup"):
        lookup_fixture(g, "lookup_small")
    if want("decode"):
        decode_fixture(g, tiny, "decode_small")
    if want("multi"):
        gm = gen_sphere_sdf(SphereSpec(center=(512, 512, 512), radius=12.0, voxel_size=1.0,
                                       half_width=3.0))
        decode_fixture(gm, tiny, "decode_multi")
    if want("train"):
        cfg = TrainConfig(l1_net=(2, 16), l0_net=(2, 32), voxel_net=(2, 32), tile_net=None,
                          ffm_size=16, ffm_scale=5.0, max_epochs=6, batch_size=4096, seed=5)
        train_fixture(g, cfg)
    if args.c1 and want("c1"):
        c1_fixture(args.c1)
    if want("procgen"):
        procgen_fixture()


def procgen_fixture():
    """Small torus (gen_torus_sdf) for the vectorized generator's parity test."""
    from svcodec.procgen import gen_torus_sdf
    g = gen_torus_sdf(16.0, 7.0, 1.0, 3.0, center=(40.0, 40.0, 20.0))
    save("procgen_torus", **grid_to_arrays(DenseLeafGrid.from_svcodec(g)))


if __name__ == "__main__":
    main()
