import cProfile, pstats, os, sys, torch
sys.path.insert(0, os.getcwd())
from bench import accept_config, make_grid, train_container
from paper_2208_04448_b200.decoder import decode_full
dev = torch.device("cuda:0")
c = train_container(make_grid("c2"), accept_config(), dev, [])
for _ in range(10): decode_full(c, dev)
torch.cuda.synchronize()
pr = cProfile.Profile(); pr.enable()
for _ in range(20): decode_full(c, dev)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(28)
