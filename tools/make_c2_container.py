"""Writes the C2 bench container as a fixture for the reference arm.

The reference arm of bench.py times the UNMODIFIED svcodec decode on the
box's CPU cores; svcodec cannot train the C2 nets in a bench's time budget
(hours of CPU), so it decodes the container the GPU arm trains: the C2 torus
512^3 encoded with ACCEPT_CONFIG by ``bench.train_container`` (deterministic:
fixed seeds, fixed-order reductions), written with svcodec's own
``write_container`` at 16-bit precision with its lossless stage.

    python tools/make_c2_container.py [out.nvdb]
"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
for p in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
    if os.path.isdir(os.path.join(p, "svcodec")):
        sys.path.append(p)
        break
from bench import accept_config, make_grid, train_container  # noqa: E402


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "tests", "golden", "c2_torus512.nvdb")
    from svcodec.config import TrainConfig
    from svcodec.container import write_container
    cfg = accept_config()
    c = train_container(make_grid("c2"), cfg, torch.device("cuda:0"), [])
    c.weight_precision = 16
    c.config = TrainConfig(**{k: getattr(cfg, k) for k in TrainConfig.__dataclass_fields__})
    write_container(c, out, lossless_stage=True)
    print(out, os.path.getsize(out), "bytes")


if __name__ == "__main__":
    main()
