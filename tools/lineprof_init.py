"""Per-line wall time of DeviceModel.__init__ on the C2 container (diagnostic)."""
import collections
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import accept_config, make_grid, train_container  # noqa: E402
from paper_2208_04448_b200 import decoder as D  # noqa: E402
from paper_2208_04448_b200 import netset as N  # noqa: E402

dev = torch.device("cuda:0")
c = train_container(make_grid("c2"), accept_config(), dev, [])
for _ in range(3):
    D.DeviceModel(c, dev)
torch.cuda.synchronize()
codes = {D.DeviceModel.__init__.__code__: "init", N.DeviceNetSet.__init__.__code__: "netset"}
acc = collections.Counter()
state = {}


def tr(frame, ev, arg):
    name = codes.get(frame.f_code)
    if name is None:
        return None

    def lt(frame, ev, arg):
        now = time.perf_counter()
        k = state.get(name)
        if k is not None:
            acc[(name, k[0])] += now - k[1]
        state[name] = (frame.f_lineno, time.perf_counter()) if ev == "line" else None
        return lt
    return lt


for _ in range(5):
    sys.settrace(tr)
    m = D.DeviceModel(c, dev)
    sys.settrace(None)
    state.clear()
for (n, ln), t in acc.most_common(15):
    print(n, ln, f"{t / 5 * 1e3:.2f} ms")
