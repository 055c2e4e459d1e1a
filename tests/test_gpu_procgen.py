"""GPU fBm density generator (nvdb_fbm_leaves) vs the reference's
gen_fbm_density (procgen.py:283-309): grids bit-identical, fixture from
tests/golden/make_golden_fbm.py."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2208_04448_b200.model import grid_from_arrays  # noqa: E402
from paper_2208_04448_b200.procgen import fbm_density  # noqa: E402


@pytest.mark.parametrize("key", ["a", "b"])
def test_fbm_density_matches_reference(golden, key):
    z = golden("procgen_fbm")
    lac, gain, f0, thr, vs = (float(v) for v in z[key + "_spec_f"])
    oc, seed, *dom = (int(v) for v in z[key + "_spec_i"])
    got = fbm_density(octaves=oc, lacunarity=lac, gain=gain, base_frequency=f0, seed=seed,
                      domain=(tuple(dom[:3]), tuple(dom[3:])), threshold=thr, voxel_size=vs)
    ref = grid_from_arrays(z, key + "_")
    for k in ("l2_origins", "l2_child", "l2_active", "l1_origins", "l1_child", "l1_active", "leaf_origins",
              "leaf_active"):
        np.testing.assert_array_equal(getattr(got, k), getattr(ref, k), err_msg=k)
    np.testing.assert_array_equal(got.leaf_values.view(np.uint32), ref.leaf_values.view(np.uint32))
    assert got.grid_class == ref.grid_class and got.background == ref.background
    print(f"{key}: {got.leaf_origins.shape[0]} leaves, {int(got.leaf_active.sum())} active voxels")
