import cProfile, pstats, sys, time, os
sys.path.insert(0, os.getcwd())
import torch
from bench import accept_config
from paper_2208_04448_b200.encoder import encode
from paper_2208_04448_b200.procgen import sphere_sdf
dev = torch.device("cuda:0")
g = sphere_sdf((256.0, 256.0, 256.0), 200.0, 1.0, 3.0)
encode(g, accept_config(), device=dev)
pr = cProfile.Profile(); pr.enable()
t = time.perf_counter(); encode(g, accept_config(), device=dev); torch.cuda.synchronize(); print("encode s", time.perf_counter() - t)
pr.disable(); pstats.Stats(pr).sort_stats("tottime").print_stats(14)
