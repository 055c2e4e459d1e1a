"""Reference quality of an 8-expert encode (sphere r 30 at (512,512,512),
tiny nets) for tests/test_gpu_train.py::test_multi_expert_encode_decode_on_gpu,
of a FOG (fBm density) encode for test_fog_encode_decode_on_gpu, and of a
3-frame warm-started sequence for test_sequence_matches_reference, and of
an fBm grid with active level-1 tiles (tile regressor path) for
test_active_tiles_match_reference.

    PYTHONPATH=/root/reference/pkg/src:/root/repo PYTHONDONTWRITEBYTECODE=1 \\
    OPENBLAS_NUM_THREADS=8 python tests/golden/make_golden_multi_encode.py

Runs the reference's own encode + decode_full on its own sphere grid with the
same TrainConfig and writes tests/golden/multi_encode.npz: the reference's
IoU against the truth, its expert count and value errors on common actives.
"""
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, os.path.dirname(HERE))

from svcodec.config import TrainConfig  # noqa: E402
from svcodec.decoder import decode_full  # noqa: E402
from svcodec.encoder import encode, encode_sequence  # noqa: E402
from svcodec.procgen import FbmSpec, SphereSpec, gen_fbm_density, gen_sphere_sdf  # noqa: E402

from paper_2208_04448_b200.model import DenseLeafGrid  # noqa: E402

CFG = dict(subdomain_size=512, l1_net=(2, 8), tile_net=None, l0_net=(2, 32), voxel_net=(2, 32),
           activation="sine", frequency=3.0, ffm_scale=5.0, ffm_size=32, lr=1e-3, decay=0.975, interval=100.0,
           max_epochs=60, sample_interval=1, batch_size=4096, seed=11)


def iou(a: DenseLeafGrid, b: DenseLeafGrid) -> float:
    def vox(g):
        li, vi = np.nonzero(g.leaf_active)
        off = np.stack([vi >> 6, (vi >> 3) & 7, vi & 7], 1)
        return set(map(tuple, (g.leaf_origins[li] + off).tolist()))
    A, B = vox(a), vox(b)
    return len(A & B) / max(1, len(A | B))


if __name__ == "__main__":
    t0 = time.time()
    g = gen_sphere_sdf(SphereSpec(center=(512.0, 512.0, 512.0), radius=30.0, voxel_size=1.0, half_width=3.0))
    c = encode(g, TrainConfig(**CFG))
    d = decode_full(c)
    truth, dec = DenseLeafGrid.from_svcodec(g), DenseLeafGrid.from_svcodec(d)
    i = iou(truth, dec)
    print(f"reference: {len(c.experts)} experts, IoU {i:.5f}, {time.time() - t0:.0f} s")
    # FOG: fBm density on a 40^3 box (FOG class: no tiles, value scale 1, no clip)
    t0 = time.time()
    fog = gen_fbm_density(FbmSpec(octaves=3, lacunarity=2.0, gain=0.5, base_frequency=0.06, seed=4,
                                  domain=((0, 0, 0), (40, 40, 40)), threshold=0.5, voxel_size=1.0))
    cf = encode(fog, TrainConfig(**CFG))
    df = decode_full(cf)
    ftruth, fdec = DenseLeafGrid.from_svcodec(fog), DenseLeafGrid.from_svcodec(df)
    fi = iou(ftruth, fdec)
    print(f"reference FOG: {len(cf.experts)} experts, IoU {fi:.5f}, {time.time() - t0:.0f} s")
    # sequence: 3 frames of a sphere moving 1 voxel per frame (the GPU tests' _moving_sphere/_seq_cfg)
    t0 = time.time()
    frames = [gen_sphere_sdf(SphereSpec(center=(20.0 + t, 20.0, 20.0), radius=11.0, voxel_size=1.0,
                                        half_width=3.0)) for t in range(3)]
    scfg = TrainConfig(l1_net=(2, 8), l0_net=(2, 16), voxel_net=(2, 24), tile_net=None, ffm_size=24,
                       max_epochs=300, batch_size=4096, lr=1e-3, refine_lr=2e-4, seed=13)
    conts, reps = encode_sequence(frames, scfg)
    seq_ep = [int(r.epochs) for r in reps]
    seq_iou = [iou(DenseLeafGrid.from_svcodec(f), DenseLeafGrid.from_svcodec(decode_full(cc)))
               for f, cc in zip(frames, conts)]
    print(f"reference sequence: epochs {seq_ep} cold {reps[0].detail.get('cold_epochs')} IoU "
          f"{np.round(seq_iou, 5)}, {time.time() - t0:.0f} s")
    # active level-1 tiles on an fBm grid: the tile regressor's decoded values
    from helpers import add_active_tiles  # noqa: E402
    t0 = time.time()
    base = gen_fbm_density(FbmSpec(octaves=3, lacunarity=2.0, gain=0.5, base_frequency=0.06, seed=4,
                                   domain=((0, 0, 0), (40, 40, 40)), threshold=0.5, voxel_size=1.0))
    tg = add_active_tiles(DenseLeafGrid.from_svcodec(base))
    tcfg = dict(CFG, tile_net=(2, 16), max_epochs=120)
    ct = encode(tg.to_svcodec(), TrainConfig(**tcfg))
    dt = DenseLeafGrid.from_svcodec(decode_full(ct))
    sel = tg.l1_active & ~tg.l1_child
    assert np.array_equal(dt.l1_origins, tg.l1_origins)
    tile_ref = dt.l1_tiles[sel]
    tile_err = float(np.sqrt(np.mean((tile_ref - tg.l1_tiles[sel]) ** 2)))
    print(f"reference tiles: {int(sel.sum())} active tiles, tile rms err vs truth {tile_err:.4f}, "
          f"tile net epochs {ct.experts[0].tile_regressor.epochs}, {time.time() - t0:.0f} s")
    np.savez_compressed(os.path.join(HERE, "multi_encode.npz"), iou=np.array([i]),
                        experts=np.array([len(c.experts)]), fog_iou=np.array([fi]),
                        seq_epochs=np.array(seq_ep), seq_iou=np.array(seq_iou),
                        seq_cold=np.array([float(reps[0].detail.get("cold_epochs", 0))]),
                        tile_ref=tile_ref.astype(np.float32), tile_err=np.array([tile_err]),
                        tile_epochs=np.array([ct.experts[0].tile_regressor.epochs]))
