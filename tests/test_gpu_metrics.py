"""GPU verification metrics against the reference's
svcodec.metrics (metrics.py:116-230) and the numpy port: IoU (SDF occupied
set with tile extents; FOG active sets with active tiles), RMSE over the
active union, mCD at zero crossings.  Counts are exact, so IoU must agree to
round-off; RMSE / mCD are f64 sums in a different order (rtol 1e-9)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from helpers import add_active_tiles  # noqa: E402
from paper_2208_04448_b200 import metrics as gm  # noqa: E402
from paper_2208_04448_b200.decoder import DeviceModel  # noqa: E402
from paper_2208_04448_b200.model import container_from_arrays  # noqa: E402


def _c1_pair(golden):
    from paper_2208_04448_b200.procgen import sphere_sdf
    truth = sphere_sdf((63.5, 63.5, 63.5), 61.0, 1.0, 3.0)
    m = DeviceModel(container_from_arrays(golden("c1_sphere128")))
    dec = m.decode(True).to_grid()
    m.close()
    return truth, dec


def test_sdf_metrics_match_port_and_reference(golden):
    from oracle.metrics_port import iou_sdf, mcd
    truth, dec = _c1_pair(golden)
    r = gm.compare(truth, dec)
    assert abs(r["iou"] - iou_sdf(truth, dec)) < 1e-12
    assert abs(r["mcd"] - mcd(truth, dec)) <= 1e-9 * mcd(truth, dec)
    print(f"C1 decode vs truth on the GPU: IoU {r['iou']:.6f}, RMSE {r['rmse']:.5f}, mCD {r['mcd']:.5f}, "
          f"surface points {r['surface_points']}")
    sm = pytest.importorskip("svcodec.metrics")
    a, b = truth.to_svcodec(), dec.to_svcodec()
    assert abs(r["iou"] - sm.iou(a, b)) < 1e-12
    assert abs(r["rmse"] - sm.rmse(a, b)) <= 1e-9 * sm.rmse(a, b)
    assert abs(r["mcd"] - sm.mcd(a, b)) <= 1e-9 * sm.mcd(a, b)
    assert gm.compare(truth, truth)["iou"] == 1.0 and gm.compare(truth, truth)["rmse"] == 0.0


def test_fog_metrics_with_active_tiles_match_reference():
    sm = pytest.importorskip("svcodec.metrics")
    from paper_2208_04448_b200.procgen import fbm_density
    a = fbm_density(octaves=3, lacunarity=2.0, gain=0.5, base_frequency=0.06, seed=4,
                    domain=((0, 0, 0), (48, 48, 48)), threshold=0.5, voxel_size=1.0, device="cuda:0")
    b = add_active_tiles(a)
    rng = np.random.default_rng(2)
    b.leaf_active = b.leaf_active ^ (rng.random(b.leaf_active.shape) < 0.03)
    b.leaf_values = (b.leaf_values + rng.normal(0, 0.05, b.leaf_values.shape)).astype(np.float32)
    r = gm.compare(a, b, mcd=False)
    ra, rb = a.to_svcodec(), b.to_svcodec()
    assert abs(r["iou"] - sm.iou(ra, rb)) < 1e-12
    assert abs(r["rmse"] - sm.rmse(ra, rb)) <= 1e-9 * sm.rmse(ra, rb)
    assert abs(gm.iou(b, a) - sm.iou(rb, ra)) < 1e-12


def test_sdf_metrics_with_tiles_and_negative_coordinates():
    """Non-positive level-1 / level-2 tiles (interior of a large sphere) enter
    the SDF occupied set as whole extents (metrics.py:68-105)."""
    sm = pytest.importorskip("svcodec.metrics")
    from paper_2208_04448_b200.procgen import sphere_sdf
    a = sphere_sdf((-20.0, 10.0, 140.0), 90.0, 1.0, 3.0)
    b = sphere_sdf((-19.0, 10.0, 140.0), 90.5, 1.0, 3.0)
    assert (a.l1_tiles[~a.l1_child] <= 0).any()
    r = gm.compare(a, b)
    ra, rb = a.to_svcodec(), b.to_svcodec()
    assert abs(r["iou"] - sm.iou(ra, rb)) < 1e-12
    assert abs(r["rmse"] - sm.rmse(ra, rb)) <= 1e-9 * sm.rmse(ra, rb)
    assert abs(r["mcd"] - sm.mcd(ra, rb)) <= 1e-9 * sm.mcd(ra, rb)
