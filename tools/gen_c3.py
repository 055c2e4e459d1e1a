"""C3 input: fBm density 1024^3, octaves 5, base frequency
4/1024, seed 9, threshold 0.45, generated on the GPU (nvdb_fbm_leaves)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2208_04448_b200.procgen import fbm_density  # noqa: E402

size = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
torch.cuda.synchronize()
t0 = time.perf_counter()
g = fbm_density(octaves=5, lacunarity=2.0, gain=0.5, base_frequency=4.0 / 1024.0, seed=9,
                domain=((0, 0, 0), (size, size, size)), threshold=0.45)
t1 = time.perf_counter()
na = int(g.leaf_active.sum())
print(f"fbm {size}^3: {g.leaf_origins.shape[0]} leaves, {na} active voxels "
      f"({100.0 * na / size ** 3:.1f} %), {g.l1_origins.shape[0]} level-1 nodes, {t1 - t0:.2f} s")
