"""C2 trainers (l1, l0, voxel; ACCEPT_CONFIG): sequential on all SMs vs each
alone on an SM share (nvdb_trainer_set_ctas) vs two nets on two streams at
once, 128 epochs each, device-timed (diagnostic; measured round 2: two
ACCEPT nets on 74 SMs each 26 ms vs 31 ms one after another on all SMs)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import accept_config, make_grid  # noqa: E402
from paper_2208_04448_b200.encoder import (DeviceTrainer, decompose, gather_expert_data, init_mlp,  # noqa: E402
                                           net_spec, stable_seed, value_scale_of, NET_TAGS)
from paper_2208_04448_b200.model import Activation, FourierFeatures  # noqa: E402

dev = torch.device("cuda:0")
cfg = accept_config()
cfg.max_epochs = int(sys.argv[1]) if len(sys.argv) > 1 else 128
g = make_grid("c2")
sub = decompose(g, cfg.subdomain_size).subdomains[0]
data = gather_expert_data(g, sub, value_scale_of(g))
sets = {"l1": (data.l1_inputs, data.l1_labels), "l0": (data.l0_inputs, data.l0_labels),
        "voxel": (data.vox_inputs, data.vox_targets)}


def make():
    out = []
    for tag, (x, y) in sets.items():
        spec = net_spec(tag, cfg)
        tid = NET_TAGS[tag]
        ff = FourierFeatures(spec.m, cfg.ffm_scale, stable_seed(cfg.seed, 0, tid, 0))
        p0 = init_mlp(2 * spec.m, [spec.arch[1]] * spec.arch[0], spec.out_dim, Activation("sine", 3.0), spec.head,
                      stable_seed(cfg.seed, 0, tid, 1))
        sampled = (not spec.full_batch) and x.shape[0] > cfg.batch_size
        out.append(DeviceTrainer(p0, ff, x, y, spec.loss_kind, cfg, cfg.lr, stable_seed(cfg.seed, 0, tid, 2),
                                 sampled, -1.0, dev))
    return out


def timed(fn):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1), 1e3 * (time.perf_counter() - t0)


trs = make()
print("sequential, all SMs:", [timed(t.run) for t in trs])
for t in trs:
    t.close()
trs = make()
w = np.asarray([t.epoch_work() for t in trs])
share = np.maximum(1, np.floor(148 * w / w.sum())).astype(int)
print("shares", share.tolist())
res = []
for t, c in zip(trs, share):
    t.set_ctas(int(c))
    res.append(timed(t.run))
print("alone on share:", res)
for t in trs:
    t.close()

# raw concurrency probes: l0 + voxel, 74 CTAs each, one enqueue of all epochs each
def probe(same_stream: bool, ctas: int = 74):
    trs = make()[1:]
    for t in trs:
        t.set_ctas(ctas)
    ss = [torch.cuda.Stream(dev) for _ in trs]
    if same_stream:
        ss = [ss[0]] * len(trs)
    cur = torch.cuda.current_stream(dev)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for s in ss:
        s.wait_stream(cur)
    for t, s in zip(trs, ss):
        with torch.cuda.stream(s):
            t._enqueue(cfg.max_epochs, s.cuda_stream)
    for s in ss:
        cur.wait_stream(s)
    e1.record()
    e1.synchronize()
    r = e0.elapsed_time(e1)
    for t in trs:
        t.close()
    return r


print("probe 2 nets x 74 CTAs, two streams:", probe(False), " one stream:", probe(True),
      " two streams 148 CTAs each:", probe(False, 148))
