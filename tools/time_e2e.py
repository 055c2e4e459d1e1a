"""decode_full (host container -> host grid) split into its phases, median of 10 (diagnostic)."""
import os
import statistics
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import accept_config, make_grid, train_container  # noqa: E402
from paper_2208_04448_b200.decoder import DeviceModel  # noqa: E402

dev = torch.device("cuda:0")
c = train_container(make_grid(os.environ.get("WORKLOAD", "c2")), accept_config(), dev, [])
ph = {"init": [], "decode": [], "to_grid": [], "total": []}
g = None
for i in range(13):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    m = DeviceModel(c, dev)
    t1 = time.perf_counter()
    d = m.decode(True)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    g = d.to_grid()
    t3 = time.perf_counter()
    if i >= 3:
        for k, v in zip(ph, (t1 - t0, t2 - t1, t3 - t2, t3 - t0)):
            ph[k].append(v * 1e3)
print({k: round(statistics.median(v), 2) for k, v in ph.items()}, "ms")
from paper_2208_04448_b200.decoder import decode_full  # noqa: E402
for pf in (False, True):
    ts = []
    for i in range(13):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        m = DeviceModel(c, dev)
        g = m.decode(True, prefetch_host=pf).to_grid()
        ts.append(time.perf_counter() - t0)
    print(f"prefetch_host={pf}: {1e3 * statistics.median(ts[3:]):.2f} ms")
ts = []
for i in range(13):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    g = decode_full(c, dev)
    ts.append(time.perf_counter() - t0)
print(f"decode_full {1e3 * statistics.median(ts[3:]):.2f} ms = {g.leaf_values.size / statistics.median(ts[3:]) / 1e9:.3f} G voxels/s")
