"""C2 training time per net (ACCEPT_CONFIG, 800 epochs), device-timed (diagnostic)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import accept_config, make_grid, train_container  # noqa: E402

g = make_grid("c2")
for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    tim = []
    train_container(g, accept_config(), torch.device("cuda:0"), tim)
    print(f"total {sum(t['ms'] for t in tim):.1f} ms:", " ".join(f"{t['tag']} {t['ms']:.1f}ms/{t['epochs']}ep loss {t['loss']:.3e}" for t in tim))
