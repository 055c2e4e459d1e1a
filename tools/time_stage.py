"""Time one decode-stage launch of mlp_eval_kernel on C2 (diagnostic).

    [NVDB_DEBUG_EVAL=..] [NVDB_DEBUG_ACT=..] python tools/time_stage.py [l0|voxel]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import accept_config, make_grid, train_container  # noqa: E402
from paper_2208_04448_b200 import _lib  # noqa: E402
from paper_2208_04448_b200.decoder import DeviceModel  # noqa: E402

stage = sys.argv[1] if len(sys.argv) > 1 else "l0"
dev = torch.device("cuda:0")
c = train_container(make_grid(os.environ.get("WORKLOAD", "c2")), accept_config(), dev, [])
m = DeviceModel(c, dev)
d = m.decode(True)
torch.cuda.synchronize()
lo = d.leaf_origins
n = lo.shape[0] * 512
out = torch.empty(n, dtype=torch.uint8, device=dev)
run = lambda: m.evaluate("l0", _lib.SRC_LEAF_VOX, lo, n, _lib.OUT_L0ACTIVE, u8=out)  # noqa: E731
for k in ("NVDB_DEBUG_EVAL", "NVDB_DEBUG_ACT"):  # diagnostics apply to the timed launches only
    if os.environ.get("TS_" + k):
        os.environ[k] = os.environ["TS_" + k]
for _ in range(3):
    run()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ts = []
for _ in range(5):
    e0.record()
    run()
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print(f"{stage} dbg {os.environ.get('NVDB_DEBUG_EVAL', '')} act {os.environ.get('NVDB_DEBUG_ACT', '')}: "
      f"{min(ts):.3f} ms  ({n} points)")
