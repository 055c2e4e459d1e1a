"""cProfile of the public decode_full (host container -> host grid) on C2."""
import cProfile
import os
import pstats
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import accept_config, make_grid, train_container  # noqa: E402
from paper_2208_04448_b200.decoder import decode_full  # noqa: E402

dev = torch.device("cuda:0")
c = train_container(make_grid(os.environ.get("WORKLOAD", "c2")), accept_config(), dev, [])
for _ in range(4):
    decode_full(c, dev)
torch.cuda.synchronize()
t0 = time.perf_counter()
g = decode_full(c, dev)
torch.cuda.synchronize()
print("decode_full s", time.perf_counter() - t0)
pr = cProfile.Profile()
pr.enable()
g = decode_full(c, dev)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(30)
