"""Run a few epochs of one ACCEPT-shaped net on C2 data (for ncu captures)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import accept_config, make_grid  # noqa: E402
from paper_2208_04448_b200.encoder import (DeviceTrainer, decompose, gather_expert_data, init_mlp,  # noqa: E402
                                           net_spec, stable_seed, value_scale_of)
from paper_2208_04448_b200.model import Activation, FourierFeatures  # noqa: E402

tag = sys.argv[1] if len(sys.argv) > 1 else "voxel"
epochs = int(sys.argv[2]) if len(sys.argv) > 2 else 6
cfg = accept_config()
g = make_grid("c2")
sub = decompose(g, 512).subdomains[0]
d = gather_expert_data(g, sub, value_scale_of(g))
x, y = {"l1": (d.l1_inputs, d.l1_labels), "l0": (d.l0_inputs, d.l0_labels),
        "voxel": (d.vox_inputs, d.vox_targets)}[tag]
spec = net_spec(tag, cfg)
ff = FourierFeatures(spec.m, cfg.ffm_scale, stable_seed(cfg.seed, 0, 3, 0))
p0 = init_mlp(2 * spec.m, [spec.arch[1]] * spec.arch[0], spec.out_dim, Activation("sine", 3.0), spec.head, 1)
tr = DeviceTrainer(p0, ff, x, y, spec.loss_kind, cfg, cfg.lr, 7, not spec.full_batch, -1.0, torch.device("cuda:0"))
tr.run(epochs)
torch.cuda.synchronize()
print("done", tr.status()[:2])
