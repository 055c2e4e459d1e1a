"""Host-side cost of the pieces of DeviceModel / decode_full on C2 (diagnostic)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import accept_config, make_grid, train_container  # noqa: E402
from paper_2208_04448_b200.decoder import DeviceModel  # noqa: E402
from paper_2208_04448_b200.netset import DeviceNetSet  # noqa: E402

dev = torch.device("cuda:0")
c = train_container(make_grid("c2"), accept_config(), dev, [])
ex = sorted(c.experts, key=lambda e: e.id)
print("patches l1", sum(len(e.patches.l1) for e in ex), "l0", sum(len(e.patches.l0) for e in ex),
      "negfill", len(c.upper_tree.leaf_negative_fill), "l1 tiles", sum(len(d) for d in c.upper_tree.l1_tiles.values()))
for _ in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ns = DeviceNetSet(ex, c.layout.size, c.layout.halo)
    t1 = time.perf_counter()
    ns.close()
    t2 = time.perf_counter()
    m = DeviceModel(c, dev)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    d = m.decode(True)
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    g = d.to_grid()
    t5 = time.perf_counter()
    m.close()
    t6 = time.perf_counter()
    print(f"netset {1e3*(t1-t0):.1f} close {1e3*(t2-t1):.1f} model {1e3*(t3-t2):.1f} decode {1e3*(t4-t3):.1f} "
          f"to_grid {1e3*(t5-t4):.1f} close {1e3*(t6-t5):.1f} ms")
