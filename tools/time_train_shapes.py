"""Device training throughput per net shape (diagnostic): sampled batches of
65,536 from 2 M random points, a fixed number of epochs (no early stop),
device-timed; prints TFLOP/s with the SURVEY.md §8(d) train flops per sample
2*(3*sum MAC - MAC_0).

    python tools/time_train_shapes.py [epochs]
"""
import json
import os
import sys
from types import SimpleNamespace

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2208_04448_b200.encoder import DeviceTrainer, init_mlp  # noqa: E402
from paper_2208_04448_b200.model import Activation, FourierFeatures  # noqa: E402

SHAPES = {  # name: (depth, width, m, omega, ffm scale)
    "accept_3x96_m192": (3, 96, 192, 3.0, 5.0),
    "accept_l1_3x48_m96": (3, 48, 96, 3.0, 5.0),
    "dragon_3x128_m256": (3, 128, 256, 1.5, 10.0),
    "leveque_3x192_m192": (3, 192, 192, 1.5, 2.0),
    "chameleon_3x256_m256": (3, 256, 256, 3.0, 10.0),
}


def train_flops(layers):
    macs = [w.shape[0] * w.shape[1] for w, _ in layers]
    return 2 * (3 * sum(macs) - macs[0])


def main():
    epochs = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    only = sys.argv[2].split(",") if len(sys.argv) > 2 else list(SHAPES)
    dev = torch.device("cuda:0")
    rng = np.random.default_rng(0)
    n = 2_000_000
    x = rng.uniform(0.05, 0.95, (n, 3)).astype(np.float32)
    y = (np.sin(6 * x[:, 0]) * np.cos(5 * x[:, 1]) * 0.5).astype(np.float32)
    out = {}
    for name in only:
        depth, width, m, omega, scale = SHAPES[name]
        cfg = SimpleNamespace(max_epochs=epochs, decay=0.975, interval=100.0, sample_interval=1, batch_size=65536)
        ff = FourierFeatures(m, scale, 11)
        p0 = init_mlp(2 * m, [width] * depth, 1, Activation("sine", omega), "linear", 12)
        tr = DeviceTrainer(p0, ff, x, y, "mse", cfg, 1e-3, 13, True, 0.0, dev,
                           path=int(os.environ.get("NVDB_TRAIN_PATH", "0")))
        tr.run(8)  # warm
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        loss, ep = tr.run()
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1)
        k = ep - 8
        fl = train_flops(p0.layers)
        tf = fl * 65536 * k / (ms * 1e-3) / 1e12
        out[name] = {"epochs": k, "ms": round(ms, 2), "us_per_epoch": round(1e3 * ms / k, 1),
                     "samples_per_s": 65536 * k / (ms * 1e-3), "tflops": round(tf, 1), "loss": loss,
                     "flops_per_sample": fl}
        print(name, json.dumps(out[name]), flush=True)
        tr.close()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
