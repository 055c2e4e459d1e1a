"""Multi-process (gloo, world_size 2, CPU) tests of the data-parallel host logic.

The GPU code paths use the same decompositions:
* training: every rank draws the same batch, takes the tile range
  ``encoder.shard_of``, sums its gradients, the sums are all-reduced and every
  rank applies the identical Adam step (DeviceTrainer with a process group);
* decode: the node-ordered leaf list is split with ``decoder.shard_range``,
  each rank decodes its range, no collective on the data path.
Here the per-rank compute is the CPU oracle, the collectives are real gloo.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, fn_name, q):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, globals()[fn_name](rank, world)))
    except Exception as exc:  # noqa: BLE001
        q.put((rank, exc))
    finally:
        dist.destroy_process_group()


def _spawn(fn_name, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, fn_name, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    for r, v in out.items():
        if isinstance(v, Exception):
            raise v
    return out


def _dp_train(rank, world):
    import torch
    import oracle as O
    from paper_2208_04448_b200.encoder import init_mlp, shard_of
    from paper_2208_04448_b200.model import Activation, FourierFeatures
    rng = np.random.default_rng(3)
    n = 1000
    x = rng.uniform(0, 1, (n, 3)).astype(np.float32)
    y = rng.uniform(-1, 1, n).astype(np.float32)
    ff = FourierFeatures(16, 5.0, 21)
    p = init_mlp(32, [32, 32], 1, Activation("sine", 3.0), "linear", 22)
    st = O.TrainState(p.layers, "sine", 3.0, ff)
    ntiles = (n + 127) // 128
    t0, t1 = shard_of(ntiles, rank, world)
    lo, hi = t0 * 128, min(n, t1 * 128)
    losses = []
    for step in range(4):
        loss, gW, gb = O.compute_grads(st, x[lo:hi], y[lo:hi], "mse", n_total=n)
        for g in list(gW) + list(gb):
            t = torch.from_numpy(np.ascontiguousarray(g))
            dist.all_reduce(t)
            g[...] = t.numpy()
        lt = torch.tensor([loss * (hi - lo)], dtype=torch.float64)
        dist.all_reduce(lt)
        losses.append(float(lt.item()) / n)
        O.adam_apply(st, gW, gb, np.float32(1e-3))
    return [w.copy() for w, _ in st.layers_interleaved()], losses


def test_data_parallel_training_matches_full_batch():
    import oracle as O
    from paper_2208_04448_b200.encoder import init_mlp
    from paper_2208_04448_b200.model import Activation, FourierFeatures
    out = _spawn("_dp_train")
    (w0, l0), (w1, l1) = out[0], out[1]
    for a, b in zip(w0, w1):
        np.testing.assert_array_equal(a, b)  # identical update on every rank
    rng = np.random.default_rng(3)
    n = 1000
    x = rng.uniform(0, 1, (n, 3)).astype(np.float32)
    y = rng.uniform(-1, 1, n).astype(np.float32)
    ff = FourierFeatures(16, 5.0, 21)
    p = init_mlp(32, [32, 32], 1, Activation("sine", 3.0), "linear", 22)
    st = O.TrainState(p.layers, "sine", 3.0, ff)
    ref_losses = [O.train_step(st, x, y, "mse", np.float32(1e-3)) for _ in range(4)]
    np.testing.assert_allclose(l0, ref_losses, rtol=1e-5)
    for a, (b, _) in zip(w0, st.layers_interleaved()):
        np.testing.assert_allclose(a, b, atol=2e-6)


def _sharded_decode(rank, world):
    import oracle as O
    from conftest import load_golden
    from paper_2208_04448_b200.decoder import shard_range
    from paper_2208_04448_b200.model import container_from_arrays
    c = container_from_arrays(load_golden("decode_multi"))
    r = O.decode(c)
    lo, hi = shard_range(r.leaf_origins.shape[0], rank, world)
    mine = (r.leaf_origins[lo:hi], r.leaf_active[lo:hi], r.leaf_values[lo:hi])
    gathered = [None] * world
    dist.all_gather_object(gathered, mine)
    return gathered


def test_sharded_decode_plan_covers_every_leaf_once():
    import oracle as O
    from conftest import load_golden
    from paper_2208_04448_b200.model import container_from_arrays
    out = _spawn("_sharded_decode")
    parts = out[0]
    full = O.decode(container_from_arrays(load_golden("decode_multi")))
    np.testing.assert_array_equal(np.concatenate([p[0] for p in parts]), full.leaf_origins)
    np.testing.assert_array_equal(np.concatenate([p[1] for p in parts]), full.leaf_active)
    np.testing.assert_array_equal(np.concatenate([p[2] for p in parts]), full.leaf_values)
    assert all(len(p[0]) > 0 for p in parts)


def test_shard_ranges_partition():
    from paper_2208_04448_b200.decoder import shard_range
    from paper_2208_04448_b200.encoder import shard_of
    for n in (0, 1, 7, 512, 12983):
        for world in (1, 2, 3, 8):
            for f in (shard_range, shard_of):
                r = [f(n, k, world) for k in range(world)]
                assert r[0][0] == 0 and r[-1][1] == n
                assert all(a[1] == b[0] for a, b in zip(r, r[1:]))
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def _gather_rows(rank, world):
    import torch
    from paper_2208_04448_b200.decoder import gather_rows
    n = 3 + 2 * rank  # unequal blocks per rank
    a = torch.arange(n * 4, dtype=torch.int32).view(n, 4) + 1000 * rank
    b = torch.full((n,), float(rank), dtype=torch.float32)
    out = gather_rows([a, b], None, dst=0)
    return None if out is None else [t.numpy() for t in out]


def test_gather_rows_concatenates_in_rank_order():
    """decoder.gather_rows (the dense-leaf / query-result gather of the sharded
    decode and query) on real gloo collectives: unequal blocks, rank order."""
    out = _spawn("_gather_rows")
    assert out[1] is None
    a, b = out[0]
    exp_a = np.concatenate([np.arange(n * 4, dtype=np.int32).reshape(n, 4) + 1000 * r
                            for r, n in ((0, 3), (1, 5))])
    np.testing.assert_array_equal(a, exp_a)
    np.testing.assert_array_equal(b, np.array([0] * 3 + [1] * 5, np.float32))
