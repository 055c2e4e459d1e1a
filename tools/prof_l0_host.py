import os, sys, time, numpy as np, torch
sys.path.insert(0, os.getcwd())
from bench import accept_config, make_grid, train_container
from paper_2208_04448_b200 import decoder as D
from paper_2208_04448_b200.model import LeafBitsMap
dev = torch.device("cuda:0")
c = train_container(make_grid("c2"), accept_config(), dev, [])
ut = c.upper_tree
for rep in range(5):
    T = [time.perf_counter()]
    l0k, l0a, l0v = D._patch_arrays([e.patches.l0 for e in c.experts], 2); T.append(time.perf_counter())
    a = l0k.astype(np.int32).reshape(-1, 3); b = np.asarray(l0a).astype(np.uint8); v = l0v.astype(np.float32); T.append(time.perf_counter())
    nf = ut.leaf_negative_fill
    norg, bits = nf.arrays(); T.append(time.perf_counter())
    nk = norg.astype(np.int32).reshape(-1, 3); nu = np.ascontiguousarray(bits).view(np.uint8).reshape(-1, 512); T.append(time.perf_counter())
    pin, buf = D._PINNED.get(nu.nbytes + (1 << 20)); buf[:nu.nbytes] = nu.reshape(-1); T.append(time.perf_counter())
    pk = np.packbits(bits, axis=1, bitorder="little"); T.append(time.perf_counter())
    m = D.DeviceModel(c, dev); T.append(time.perf_counter())
    torch.cuda.synchronize(); T.append(time.perf_counter())
    print(type(nf).__name__, len(l0k), norg.shape, " ".join(f"{1e3*(y-x):.3f}" for x, y in zip(T, T[1:])))
