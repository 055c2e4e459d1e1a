"""Host-side time of decode_full's phases on C2 (diagnostic): wall time spent
inside each wrapped method, median over 10 calls, beside the call's total."""
import functools
import os
import statistics
import sys
import time
from collections import defaultdict

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import accept_config, make_grid, train_container  # noqa: E402
from paper_2208_04448_b200 import decoder as D  # noqa: E402

dev = torch.device("cuda:0")
c = train_container(make_grid("c2"), accept_config(), dev, [])
acc = defaultdict(float)


def wrap(cls, name):
    f = getattr(cls, name)

    @functools.wraps(f)
    def g(*a, **k):
        t = time.perf_counter()
        try:
            return f(*a, **k)
        finally:
            acc[f"{cls.__name__}.{name}"] += time.perf_counter() - t
    setattr(cls, name, g)


for n in ("__init__", "_ensure_l0", "decode", "_decode_pipelined", "select", "evaluate", "_host_prefetch",
          "_upload", "_slots"):
    wrap(D.DeviceModel, n)
for n in ("to_grid", "check"):
    wrap(D.DeviceDecode, n)
rows = defaultdict(list)
for i in range(40):
    torch.cuda.synchronize()
    acc.clear()
    t0 = time.perf_counter()
    D.decode_full(c, dev)
    tot = time.perf_counter() - t0
    if i >= 20:
        rows["total"].append(tot)
        for k, v in acc.items():
            rows[k].append(v)
print("per-call totals (ms):", " ".join(f"{1e3 * v:.2f}" for v in rows["total"]))
for k, v in rows.items():
    print(f"{k:32s} {1e3 * statistics.median(v):7.3f} ms")
