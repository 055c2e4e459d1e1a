"""decode_full in the bench's loop shape (previous grid held): per-call wall
time, its DeviceModel / decode / to_grid split and the pinned-pool blocks
allocated in the call (diagnostic)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import accept_config, make_grid, train_container  # noqa: E402
from paper_2208_04448_b200 import decoder as D  # noqa: E402

dev = torch.device("cuda:0")
c = train_container(make_grid("c2"), accept_config(), dev, [])
news = []
_get = D._PinnedPool.get


def get(self, nbytes):
    n0 = len(self.blocks)
    ids = {id(b[0]) for b in self.blocks}
    t = time.perf_counter()
    r = _get(self, nbytes)
    if id(r[0]) not in ids:
        news.append((nbytes >> 20, round((time.perf_counter() - t) * 1e3, 2), n0))
    return r


D._PinnedPool.get = get
gct = []
_gc0 = [0.0]


def _gccb(phase, info):
    if phase == "start":
        _gc0[0] = time.perf_counter()
    else:
        gct.append((info["generation"], round((time.perf_counter() - _gc0[0]) * 1e3, 2)))


import gc  # noqa: E402
gc.callbacks.append(_gccb)
if os.environ.get("AFTER_QUERY"):
    import bench  # noqa: E402
    mm = D.DeviceModel(c, dev)
    bench.query_bench(mm, dev, 20, rank=0, world=1)
    if os.environ.get("AFTER_QUERY") == "pool":  # drop the pinned blocks the query section left
        D._PINNED.blocks.clear()
    if os.environ.get("AFTER_QUERY") == "mem":  # release the device memory it left cached
        del mm
        import gc as _g
        _g.collect()
        torch.cuda.empty_cache()
if os.environ.get("BIG_ALLOC"):
    big = torch.empty(int(os.environ["BIG_ALLOC"]) << 20, dtype=torch.uint8, device=dev)
g = None
for i in range(12):
    news.clear()
    gct.clear()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    m = D._as_model(c, dev)
    t1 = time.perf_counter()
    d = m.decode(True, prefetch_host=True)
    t2 = time.perf_counter()
    g = d.to_grid()
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    print(f"call {i}: total {1e3 * (t3 - t0):.2f} ms (model {1e3 * (t1 - t0):.2f}, decode {1e3 * (t2 - t1):.2f}, "
          f"to_grid {1e3 * (t3 - t2):.2f}); new pinned blocks (MiB, ms, pool size) {news}; gc {gct}", flush=True)
