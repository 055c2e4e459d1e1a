"""Pin the oracle's IoU/mCD port against the reference's recorded AC4 result.

pkg/test_output.txt:20 records IoU 0.9984 (0.99835 in SURVEY.md §4) and
mCD 0.0313 dx for the C1 container decoded by the reference; the oracle
decode of the same container (pinned in test_oracle_golden) fed to the
metric port must reproduce them.
"""
import numpy as np

import oracle as O
from oracle.metrics_port import iou_sdf, mcd
from paper_2208_04448_b200.model import container_from_arrays
from paper_2208_04448_b200.procgen import sphere_sdf


def test_ac4_metrics_reproduced(golden):
    z = golden("c1_sphere128")
    c = container_from_arrays(z)
    truth = sphere_sdf((63.5, 63.5, 63.5), 61.0, 1.0, 3.0)
    dec = O.topology_grid(c, O.decode(c))
    i = iou_sdf(truth, dec)
    d = mcd(truth, dec)
    print(f"IoU {i:.5f} mCD {d:.4f}")
    assert abs(i - 0.99835) < 5e-5
    assert abs(d - 0.0313) < 5e-4
