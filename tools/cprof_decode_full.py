"""cProfile of 20 decode_full calls on C2 (diagnostic).  BIG_ALLOC=<MiB>:
hold that much extra device memory first."""
import cProfile
import os
import pstats
import sys

import torch

sys.path.insert(0, os.getcwd())
from bench import accept_config, make_grid, train_container  # noqa: E402
from paper_2208_04448_b200.decoder import decode_full  # noqa: E402

dev = torch.device("cuda:0")
c = train_container(make_grid("c2"), accept_config(), dev, [])
if os.environ.get("BIG_ALLOC"):
    big = torch.empty(int(os.environ["BIG_ALLOC"]) << 20, dtype=torch.uint8, device=dev)
for _ in range(10):
    decode_full(c, dev)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    decode_full(c, dev)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
