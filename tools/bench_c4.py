"""C4-shaped animated sequence (BASELINE configs[3]): moving
sphere (centre (256,256,256) + t*(1,0,0), radius 200, half width 3) at 512^3,
encode_sequence with warm starts on the GPU.  Nets: the LeVeque row of PAPER.md Table 3
(SURVEY.md §8(d) C4): S = 1024, L1 3x96, L0 / voxel 3x192,
sine / 1.5, FFM 2.0 / 192, lr 0.001 / refine 0.0002, decay 0.975 / 100,
2500 epochs, B = 2^16 (layer-streamed training for the 192-wide nets).
Reports per-frame
epochs (frame 0 cold + refine, later frames warm with the frame-0 loss
targets) and the device training time.

    python tools/bench_c4.py [frames]
"""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2208_04448_b200.encoder import TrainConfig  # noqa: E402
from paper_2208_04448_b200.encoder import encode_sequence  # noqa: E402
from paper_2208_04448_b200.procgen import sphere_sdf  # noqa: E402

frames = int(sys.argv[1]) if len(sys.argv) > 1 else 4
t0 = time.perf_counter()
grids = [sphere_sdf((256.0 + t, 256.0, 256.0), 200.0, 1.0, 3.0) for t in range(frames)]
tgen = time.perf_counter() - t0
cfg = TrainConfig(subdomain_size=1024, l1_net=(3, 96), tile_net=None, l0_net=(3, 192), voxel_net=(3, 192),
                  activation="sine", frequency=1.5, ffm_scale=2.0, ffm_size=192, lr=1e-3, refine_lr=2e-4,
                  decay=0.975, interval=100.0, max_epochs=2500, sample_interval=1, batch_size=65536,
                  significance_threshold=None, strict_topology=False, seed=4242)
torch.cuda.synchronize()
t1 = time.perf_counter()
containers, reports = encode_sequence(grids, cfg, 16, 1, device=torch.device("cuda:0"))
torch.cuda.synchronize()
t2 = time.perf_counter()
print(json.dumps({"workload": f"C4-shaped: moving sphere r=200 at 512^3, {frames} frames, LeVeque nets (L1 3x96, L0/voxel 3x192/m192, 2500 epochs)",
                  "generate_s": round(tgen, 1), "encode_sequence_s": round(t2 - t1, 1),
                  "active_voxels_frame0": int(grids[0].leaf_active.sum()),
                  "frames": [{"frame": r.frame, "epochs": r.epochs, "loss": r.final_loss, **r.detail} for r in reports]}))
