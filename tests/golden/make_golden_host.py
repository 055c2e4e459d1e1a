"""Golden fixtures for the host-side training set-up, from the reference itself.

    PYTHONPATH=/root/reference/pkg/src:/root/repo PYTHONDONTWRITEBYTECODE=1 \
    python tests/golden/make_golden_host.py

neural.init_mlp (neural.py:168-185) for several shapes / activations / seeds;
partition.decompose (partition.py:74-120) and, per subdomain,
encoder._expert_norm + _gather_expert_data (encoder.py:181-235) on two grids:
a sphere straddling the 2 x 2 x 2 lattice point at 512 (8 experts, leaves in
the halo of their neighbours), a torus around a lattice line, and a small
fBm density (FOG: value scale 1).
tests/test_host_logic.py compares the framework's host code with them.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from svcodec import neural as N  # noqa: E402
from svcodec.encoder import _expert_norm, _flatten_grid, _gather_expert_data, _value_scale  # noqa: E402
from svcodec.partition import decompose  # noqa: E402
from svcodec.procgen import SphereSpec, gen_sphere_sdf  # noqa: E402

from paper_2208_04448_b200.model import DenseLeafGrid, grid_to_arrays  # noqa: E402

INIT_CASES = [  # (in_dim, hidden, out_dim, activation, frequency, head, seed)
    (384, [96, 96, 96], 1, "sine", 3.0, "linear", 11),
    (96, [48, 48, 48], 3, "sine", 3.0, "logits", 12),
    (512, [256, 256, 256], 1, "sine", 1.5, "binary", 13),
    (40, [24, 24], 1, "relu", 1.0, "linear", 14),
    (64, [100, 60], 3, "tanh", 1.0, "logits", 15),
]


def grids():
    from svcodec.procgen import FbmSpec, gen_fbm_density, gen_torus_sdf
    a = gen_sphere_sdf(SphereSpec(center=(512, 512, 512), radius=14.0, voxel_size=1.0, half_width=3.0))
    # a thin torus around the lattice line x = y = 512 (4 experts, leaves in each other's halos)
    b = gen_torus_sdf(30.0, 8.0, 1.0, 3.0, center=(512.0, 512.0, 300.0))
    f = gen_fbm_density(FbmSpec(octaves=3, lacunarity=2.0, gain=0.5, base_frequency=1.0 / 32.0, seed=4,
                                domain=((0, 0, 0), (48, 48, 48)), threshold=0.5))
    return {"straddle": a, "torus": b, "fog": f}


def main():
    out = {}
    for i, (ind, hid, od, act, fr, head, seed) in enumerate(INIT_CASES):
        p = N.init_mlp(ind, hid, od, N.Activation(act, fr), head, seed)
        for li, (w, b) in enumerate(p.layers):
            out[f"init{i}_w{li}"] = w
            out[f"init{i}_b{li}"] = b
    for name, g in grids().items():
        layout = decompose(g, 512)
        arrays = _flatten_grid(g)
        out.update(grid_to_arrays(DenseLeafGrid.from_svcodec(g), f"{name}_g_"))
        out[f"{name}_cells"] = np.array([s.cell for s in layout.subdomains], np.int64)
        out[f"{name}_clusters"] = np.array([s.cluster_id for s in layout.subdomains], np.int64)
        scale = _value_scale(g)
        for s in layout.subdomains:
            no, ns = _expert_norm(s, arrays)
            d = _gather_expert_data(g, s, arrays, scale)
            q = f"{name}_e{s.id}_"
            out[q + "norm"] = np.array([*no, ns], np.float64)
            for k in ("l1_inputs", "l1_labels", "l0_inputs", "l0_labels", "vox_inputs", "vox_targets"):
                v = getattr(d, k)
                out[q + k] = np.zeros(0) if v is None else v
    path = os.path.join(HERE, "host_setup.npz")
    np.savez_compressed(path, **out)
    print(f"host_setup: {os.path.getsize(path) / 1024:.1f} KiB")


if __name__ == "__main__":
    main()
