"""Where C3's encode() time goes (diagnostic): fBm 1024^3 on the GPU, then
one encode() with the Chameleon row under cProfile (cumulative), on 1 GPU."""
import cProfile
import os
import pstats
import sys
import time
from types import SimpleNamespace

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from c3_pipeline import CHAMELEON  # noqa: E402
from paper_2208_04448_b200.encoder import encode  # noqa: E402
from paper_2208_04448_b200.procgen import fbm_density  # noqa: E402

dev = torch.device("cuda:0")
size = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
epochs = int(sys.argv[2]) if len(sys.argv) > 2 else 2500
cfg = SimpleNamespace(**dict(CHAMELEON, max_epochs=epochs))
g = fbm_density(octaves=5, lacunarity=2.0, gain=0.5, base_frequency=4.0 / 1024.0, seed=9,
                domain=((0, 0, 0), (size, size, size)), threshold=0.45, device=dev)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
t = time.perf_counter()
c = encode(g, cfg, 16, device=dev)
torch.cuda.synchronize()
print("encode s", round(time.perf_counter() - t, 2))
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(28)
