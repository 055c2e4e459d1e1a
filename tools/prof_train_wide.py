"""A few epochs of one Table-3 shape on the layer-streamed training kernels
(for ncu launch lists / captures; diagnostic).
    python tools/prof_train_wide.py [depth width m] [epochs]"""
import os
import sys
from types import SimpleNamespace

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2208_04448_b200.encoder import DeviceTrainer, init_mlp  # noqa: E402
from paper_2208_04448_b200.model import Activation, FourierFeatures  # noqa: E402

a = [int(v) for v in sys.argv[1:]]
depth, width, m = a[:3] if len(a) >= 3 else (3, 256, 256)
epochs = a[3] if len(a) >= 4 else 6
rng = np.random.default_rng(0)
n = 2_000_000
x = rng.uniform(0.05, 0.95, (n, 3)).astype(np.float32)
y = (np.sin(6 * x[:, 0]) * np.cos(5 * x[:, 1]) * 0.5).astype(np.float32)
cfg = SimpleNamespace(max_epochs=epochs + 2, decay=0.975, interval=100.0, sample_interval=1, batch_size=65536)
ff = FourierFeatures(m, 10.0, 11)
p0 = init_mlp(2 * m, [width] * depth, 1, Activation("sine", 3.0), "linear", 12)
tr = DeviceTrainer(p0, ff, x, y, "mse", cfg, 1e-3, 13, True, 0.0, torch.device("cuda:0"))
tr.run(2)
torch.cuda.synchronize()
tr.run(epochs)
torch.cuda.synchronize()
print("done")
