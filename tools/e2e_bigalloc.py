"""Device decode and decode_full on C2 before / after holding extra device
memory (diagnostic for the e2e variance)."""
import os
import statistics
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import accept_config, make_grid, train_container  # noqa: E402
from paper_2208_04448_b200.decoder import DeviceModel, decode_full  # noqa: E402

dev = torch.device("cuda:0")
c = train_container(make_grid("c2"), accept_config(), dev, [])
m = DeviceModel(c, dev)


def measure(tag):
    ev = []
    for i in range(12):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        m.decode(True)
        e1.record()
        torch.cuda.synchronize()
        ev.append(e0.elapsed_time(e1))
    wall, allocs = [], []
    for i in range(12):
        torch.cuda.synchronize()
        s0 = torch.cuda.memory_stats(dev)
        t0 = time.perf_counter()
        decode_full(c, dev)
        torch.cuda.synchronize()
        wall.append(1e3 * (time.perf_counter() - t0))
        s1 = torch.cuda.memory_stats(dev)
        allocs.append(tuple(s1.get(k, 0) - s0.get(k, 0) for k in ("num_device_alloc", "num_device_free",
                                                                   "allocated_bytes.all.current",
                                                                   "reserved_bytes.all.current")))
    print(f"{tag}: device decode {statistics.median(ev[2:]):.2f} ms, decode_full {statistics.median(wall[2:]):.2f} ms "
          f"{[round(w, 1) for w in wall[2:]]} cudaMalloc/cudaFree/allocated/reserved delta per call {allocs[2:6]}", flush=True)


measure("base")
big = torch.empty(4 << 30, dtype=torch.uint8, device=dev)
measure("+4 GiB held")
big.zero_()
measure("+4 GiB touched")
del big
measure("released (cached)")
torch.cuda.empty_cache()
measure("released (empty_cache)")
