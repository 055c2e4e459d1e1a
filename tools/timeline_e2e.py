"""decode_full (C2) timeline from torch.profiler (CUPTI): host phases and
every kernel / copy with start and end relative to the call (diagnostic)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import accept_config, make_grid, train_container  # noqa: E402
from paper_2208_04448_b200.decoder import decode_full  # noqa: E402

dev = torch.device("cuda:0")
c = train_container(make_grid("c2"), accept_config(), dev, [])
for _ in range(5):
    decode_full(c, dev)
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CPU, torch.profiler.ProfilerActivity.CUDA]) as prof:
    with torch.profiler.record_function("decode_full"):
        decode_full(c, dev)
    torch.cuda.synchronize()
prof.export_chrome_trace("/tmp/tl.json")
ev = json.load(open("/tmp/tl.json"))["traceEvents"]
t0 = min(e["ts"] for e in ev if e.get("name") == "decode_full")
rows = []
for e in ev:
    if e.get("ph") != "X":
        continue
    cat = e.get("cat", "")
    if cat in ("kernel", "gpu_memcpy", "gpu_memset") or e.get("name") == "decode_full" or \
            (cat == "cpu_op" and e["name"].startswith("cudaStreamSynchronize")) or \
            (cat == "cuda_runtime" and "Synchronize" in e["name"]):
        rows.append((e["ts"] - t0, e["dur"], cat, e["name"][:70], e.get("args", {}).get("stream", "")))
for r in sorted(rows):
    print(f"{r[0]:9.1f} {r[1]:8.1f}  {r[2]:12s} s{r[4]!s:3s} {r[3]}")
