"""C3 end to end (BASELINE configs[2]): fBm density 1024^3
(octaves 5, base frequency 4/1024, seed 9, threshold 0.45) generated on the
GPU, encoded with the Chameleon row of PAPER.md Table 3 (L1 3x128, L0 / voxel
3x256, sine / 3.0, FFM 10 / 256, lr 1e-3, decay 0.975 / 100, 2500 epochs,
B = 2^16) at S = 512 (8 experts, 2 x 2 x 2), then decoded (level-1 stage,
patches, leaves, finalize) and compared with the input.

Under torchrun with N ranks (one per GPU) the experts train expert-parallel
(round-robin, no collective while training) and the decode splits the
leaves into N contiguous ranges; rank 0 prints one JSON line.

    python tools/c3_pipeline.py [size] [max_epochs]
    python -m torch.distributed.run --nproc-per-node 8 tools/c3_pipeline.py
"""
import json
import os
import sys
import time
from types import SimpleNamespace

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2208_04448_b200.decoder import DeviceModel  # noqa: E402
from paper_2208_04448_b200.encoder import encode  # noqa: E402
from paper_2208_04448_b200.procgen import fbm_density  # noqa: E402

CHAMELEON = dict(subdomain_size=512, l1_net=(3, 128), tile_net=None, l0_net=(3, 256), voxel_net=(3, 256),
                 activation="sine", frequency=3.0, ffm_scale=10.0, ffm_size=256, lr=1e-3, refine_lr=None,
                 decay=0.975, interval=100.0, max_epochs=2500, sample_interval=1, batch_size=65536,
                 significance_threshold=None, strict_topology=False, seed=4242)


def fwd_flops(net):
    return int(sum(2 * w.shape[0] * w.shape[1] for w, _ in net.params.layers))


def leaf_keys(o):
    o = o.to(torch.int64)
    return (o[:, 0] << 42) | (o[:, 1] << 21) | o[:, 2]


def run(size: int, epochs: int, dev, group=None) -> dict:
    """The whole C3 pipeline on this rank's GPU (all ranks of `group` call it);
    returns the result dict (times are max over ranks)."""
    import torch.distributed as dist
    world = dist.get_world_size(group) if group is not None else 1
    rank = dist.get_rank(group) if group is not None else 0
    cfg = SimpleNamespace(**dict(CHAMELEON, max_epochs=epochs))
    t0 = time.perf_counter()
    g = fbm_density(octaves=5, lacunarity=2.0, gain=0.5, base_frequency=4.0 / 1024.0, seed=9,
                    domain=((0, 0, 0), (size, size, size)), threshold=0.45, device=dev)
    torch.cuda.synchronize()
    t_gen = time.perf_counter() - t0
    if world > 1:
        dist.barrier(group)
    t0 = time.perf_counter()
    c = encode(g, cfg, 16, device=dev, group=group)
    torch.cuda.synchronize()
    t_enc = time.perf_counter() - t0
    if world > 1:
        te = torch.tensor([t_enc], dtype=torch.float64, device=dev)
        dist.all_reduce(te, op=dist.ReduceOp.MAX, group=group)
        t_enc = float(te.item())
    m = DeviceModel(c, dev)
    shard = (rank, world) if world > 1 else None
    d = m.decode(True, shard=shard)  # warm
    torch.cuda.synchronize()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    ts = []
    for _ in range(3):
        flush.random_(0, 255)
        if world > 1:
            dist.barrier(group)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        d = m.decode(True, shard=shard)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = float(np.median(ts))
    if os.environ.get("NVDB_PROFILE") == "1":  # ncu --profile-from-start off: one decode's launch list
        torch.cuda.profiler.start()
        m.decode(True, shard=shard)
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
    cnt = torch.tensor([d.leaf_count * 512, d.regressor_evaluations, ms], dtype=torch.float64, device=dev)
    if world > 1:
        mx = cnt[2:].clone()
        dist.all_reduce(cnt, group=group)
        dist.all_reduce(mx, op=dist.ReduceOp.MAX, group=group)
        cnt[2] = mx[0]
    nvox, nact, ms = int(cnt[0].item()), int(cnt[1].item()), float(cnt[2].item())
    # quality: decoded active set vs the input's (FOG: IoU over active voxels), on the device
    iou = None
    if world == 1:
        tk = leaf_keys(torch.from_numpy(g.leaf_origins).to(dev))
        order = torch.argsort(tk)
        tk = tk[order]
        ta = torch.from_numpy(g.leaf_active).to(dev)[order]
        dk = leaf_keys(d.leaf_origins)
        pos = torch.searchsorted(tk, dk).clamp(max=tk.numel() - 1)
        hit = tk[pos] == dk
        da = d.leaf_active.view(-1, 512).bool()
        inter = int((ta[pos[hit]] & da[hit]).sum().item())
        union = int(ta.sum().item()) + int(da.sum().item()) - inter
        iou = inter / max(union, 1)
    e = c.experts[0]
    F = {t: fwd_flops(n) for t, n in e.nets() if n is not None}
    epochs_run = {f"{x.id}:{t}": n.epochs for x in c.experts for t, n in x.nets() if n is not None}
    F_all = (m.n1 * 4096 * F["l1"] + nvox * F["l0"] + nact * F["voxel"])
    m.close()
    return {
            "workload": f"C3 fBm {size}^3 (545 M active at 1024^3), 8 experts at S=512, Chameleon nets "
                        f"(L1 3x128/m128, L0+voxel 3x256/m256, {epochs} epochs max), trained by encode()",
            "ranks": world, "generate_s": round(t_gen, 2), "encode_s": round(t_enc, 1),
            "leaf_voxels": nvox, "regressor_evaluations": nact, "l1_slots": m.n1 * 4096,
            "decode_ms": round(ms, 2), "decode_voxels_per_s": nvox / (ms * 1e-3),
            "decode_tflops": F_all / (ms * 1e-3) / 1e12,
            "iou_active": iou, "patches": sum(len(x.patches) for x in c.experts),
            "epochs": epochs_run}


def main():
    size = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
    epochs = int(sys.argv[2]) if len(sys.argv) > 2 else 2500
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    group = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
        group = dist.group.WORLD
    r = run(size, epochs, dev, group)
    if int(os.environ.get("RANK", "0")) == 0:
        print(json.dumps(r), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
