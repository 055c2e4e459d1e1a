"""cProfile (tottime) of DeviceModel construction on C2 (diagnostic)."""
import cProfile
import os
import pstats
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import accept_config, make_grid, train_container  # noqa: E402
from paper_2208_04448_b200.decoder import DeviceModel  # noqa: E402

dev = torch.device("cuda:0")
c = train_container(make_grid("c2"), accept_config(), dev, [])
DeviceModel(c, dev).close()
pr = cProfile.Profile()
pr.enable()
m = DeviceModel(c, dev)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
