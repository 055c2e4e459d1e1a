"""Golden fBm density grids produced by the reference's gen_fbm_density.

    PYTHONPATH=/root/reference/pkg/src:/root/repo PYTHONDONTWRITEBYTECODE=1 \\
    python tests/golden/make_golden_fbm.py

Writes tests/golden/procgen_fbm.npz: two specs (a small odd-offset domain with
3 octaves; a C3-shaped 5-octave spec on a 48^3 box) with the grids in
grid_to_arrays form under the prefixes a_ and b_, and the spec parameters.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from svcodec.procgen import FbmSpec, gen_fbm_density  # noqa: E402

from paper_2208_04448_b200.model import DenseLeafGrid, grid_to_arrays  # noqa: E402

SPECS = {
    "a": dict(octaves=3, lacunarity=2.0, gain=0.5, base_frequency=0.07, seed=9,
              domain=((-5, 3, 0), (37, 41, 30)), threshold=0.5, voxel_size=1.0),
    "b": dict(octaves=5, lacunarity=2.0, gain=0.5, base_frequency=4.0 / 64.0, seed=9,
              domain=((0, 0, 0), (48, 48, 48)), threshold=0.45, voxel_size=1.0),
}

if __name__ == "__main__":
    arrays = {}
    for k, sp in SPECS.items():
        g = gen_fbm_density(FbmSpec(**sp))
        arrays.update(grid_to_arrays(DenseLeafGrid.from_svcodec(g), k + "_"))
        arrays[k + "_spec_f"] = np.array([sp["lacunarity"], sp["gain"], sp["base_frequency"], sp["threshold"],
                                          sp["voxel_size"]])
        arrays[k + "_spec_i"] = np.array([sp["octaves"], sp["seed"], *sp["domain"][0], *sp["domain"][1]])
    path = os.path.join(HERE, "procgen_fbm.npz")
    np.savez_compressed(path, **arrays)
    print(f"procgen_fbm: {os.path.getsize(path) / 1024:.1f} KiB")
