"""decode_full wall time per call before and after the bench's query section (diagnostic)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from bench import accept_config, make_grid, train_container  # noqa: E402
from paper_2208_04448_b200.decoder import DeviceModel, decode_full  # noqa: E402

dev = torch.device("cuda:0")
c = train_container(make_grid("c2"), accept_config(), dev, [])


def run(tag, k=8):
    ts = []
    for _ in range(k):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        decode_full(c, dev)
        torch.cuda.synchronize()
        ts.append(round((time.perf_counter() - t0) * 1e3, 2))
    print(tag, ts, flush=True)


run("fresh")
m = DeviceModel(c, dev)
for _ in range(25):
    m.decode(True)
torch.cuda.synchronize()
run("after device decodes")
bench.query_bench(m, dev, 20, rank=0, world=1)
run("after query_bench")
