"""Shared test helpers: rebuild nets/configs from golden fixtures."""
from types import SimpleNamespace

import numpy as np

from paper_2208_04448_b200.model import Activation, FourierFeatures, MlpParams

ACTS = ["relu", "tanh", "sine"]
HEADS = ["linear", "logits", "binary"]
LOSSES = ["mse", "ce", "bce"]


def net_from_fixture(z, q):
    cfg = z[q + "cfg"]
    hidden = list(z[q + "hidden"])
    nl = len(hidden) + 1
    layers = [(z[q + f"w{i}"].copy(), z[q + f"b{i}"].copy()) for i in range(nl)]
    act = Activation(ACTS[int(cfg[0])], float(cfg[1]))
    ff = FourierFeatures(int(cfg[2]), float(cfg[6]) if len(cfg) == 7 else 5.0, int(cfg[5]))
    return MlpParams(layers, act, HEADS[int(cfg[4])]), ff


def tiny_cfg(**kw):
    base = dict(subdomain_size=512, l1_net=(2, 8), tile_net=None, l0_net=(2, 16),
                voxel_net=(2, 16), activation="sine", frequency=3.0, ffm_scale=5.0,
                ffm_size=16, lr=1e-3, refine_lr=None, decay=0.975, interval=100.0,
                max_epochs=40, sample_interval=1, batch_size=4096,
                significance_threshold=None, strict_topology=False, seed=11)
    base.update(kw)
    return SimpleNamespace(**base)


def add_active_tiles(g):
    """A copy of a DenseLeafGrid with active level-1 tiles added in empty
    slots (every slot with (i + j + k) % 5 == 0 that is neither a child nor
    a tile), values a smooth function of the slot centre in (0.55, 0.95):
    exercises the tile regressor path (decoder.py:136-141)."""
    import copy
    from paper_2208_04448_b200.model import L1_LOCAL
    h = copy.deepcopy(g)
    ijk = L1_LOCAL  # (4096, 3) slot index triples, idx1 order
    pick = ((ijk.sum(axis=1) % 5) == 0)[None, :] & ~h.l1_child & ~h.l1_active
    cen = h.l1_origins[:, None, :].astype(np.float64) + ijk[None] * 8.0 + 4.0
    val = (0.75 + 0.2 * np.sin(cen[..., 0] / 9.0) * np.cos(cen[..., 1] / 7.0)).astype(np.float32)
    h.l1_active = h.l1_active | pick
    h.l1_tiles = np.where(pick, val, h.l1_tiles).astype(np.float32)
    return h


# SURVEY.md §8(c) parity bars, calibrated by the survey's fp16 simulation on
# the C1 (AC4) container: regressor error vs forward_block on the same points
# in SCALED units (value / value_scale): max <= 2e-3, RMS <= 5e-4; level-0
# occupancy agreement >= 99.99 %.  GEMM operands are fp16 with fp32
# accumulation; a container's weights are compared as a 16-bit container
# stores them (container.py:241-244), so weight rounding is not an error term.
VAL_MAX_SCALED, VAL_RMS_SCALED, OCC_BAR = 2e-3, 5e-4, 0.9999


def assert_value_bars(err, scale, what=""):
    """err: |gpu - reference| in world units; scale: the container's value_scale
    (or max(1, |reference|) for raw network outputs)."""
    err = np.asarray(err, np.float64) / float(scale)
    mx = float(err.max()) if err.size else 0.0
    rms = float(np.sqrt(np.mean(err ** 2))) if err.size else 0.0
    print(f"{what} scaled error max {mx:.2e} rms {rms:.2e} (bars {VAL_MAX_SCALED:.0e} / {VAL_RMS_SCALED:.0e})")
    assert mx <= VAL_MAX_SCALED and rms <= VAL_RMS_SCALED, (what, mx, rms)


def fp16_params(params):
    """MlpParams with every weight and bias rounded to fp16 (weight_precision = 16)."""
    params.layers = [(np.asarray(w, np.float32).astype(np.float16).astype(np.float32),
                      np.asarray(b, np.float32).astype(np.float16).astype(np.float32)) for w, b in params.layers]
    return params
