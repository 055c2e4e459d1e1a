"""Train the C2 container on the GPU and pickle it to gpurun_out/ (host-side profiling aid)."""
import os
import pickle
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import accept_config, make_grid, train_container  # noqa: E402

c = train_container(make_grid(os.environ.get("WORKLOAD", "c2")), accept_config(), torch.device("cuda:0"), [])
os.makedirs("gpurun_out", exist_ok=True)
with open("gpurun_out/c2_container.pkl", "wb") as f:
    pickle.dump(c, f, protocol=pickle.HIGHEST_PROTOCOL)
print("pickled", os.path.getsize("gpurun_out/c2_container.pkl"))
