"""The vectorized generators reproduce the reference's grids exactly."""
import numpy as np
import pytest

from paper_2208_04448_b200.model import grid_from_arrays
from paper_2208_04448_b200.procgen import sphere_sdf, torus_sdf


def _same(a, b):
    for k in ("l2_origins", "l2_child", "l2_active", "l2_tiles", "l1_origins", "l1_child", "l1_active",
              "l1_tiles", "leaf_origins", "leaf_active"):
        np.testing.assert_array_equal(getattr(a, k), getattr(b, k), err_msg=k)
    np.testing.assert_array_equal(a.leaf_values.view(np.uint32), b.leaf_values.view(np.uint32))
    assert a.background == b.background and a.root_tiles == b.root_tiles


def test_sphere_matches_reference(golden):
    ref = grid_from_arrays(golden("decode_small"), "g_")
    _same(sphere_sdf((20, 20, 20), 12.0, 1.0, 3.0), ref)


def test_torus_matches_reference(golden):
    ref = grid_from_arrays(golden("procgen_torus"))
    _same(torus_sdf(16.0, 7.0, 1.0, 3.0, center=(40.0, 40.0, 20.0)), ref)
