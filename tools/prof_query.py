"""HybridGrid.query_device on the C2 container, 2^27 uniform int32 coords in
[-32, 544)^3 (the bench's query stream): per-call device time and, under
ncu, the launch list of one call (diagnostic)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import accept_config, make_grid, train_container  # noqa: E402
from paper_2208_04448_b200.decoder import make_hybrid  # noqa: E402

dev = torch.device("cuda:0")
c = train_container(make_grid("c2"), accept_config(), dev, [])
hg = make_hybrid(c, dev)
g = torch.Generator(device=dev)
g.manual_seed(0)
coords = torch.randint(-32, 544, (1 << 27, 3), dtype=torch.int32, device=dev, generator=g)
for _ in range(3):
    hg.query_device(coords)
torch.cuda.synchronize()
ts = []
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    hg.query_device(coords)
    e1.record()
    e1.synchronize()
    ts.append(e0.elapsed_time(e1))
ts.sort()
print(f"query_device {ts[len(ts) // 2]:.3f} ms = {coords.shape[0] / ts[len(ts) // 2] / 1e6:.1f} G q/s, "
      f"regressor rows {hg.regressor_evaluations // 13}")
if os.environ.get("NVDB_PROFILE") == "1":
    torch.cuda.profiler.start()
    hg.query_device(coords)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
