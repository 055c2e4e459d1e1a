"""Multi-rank paths through the public API on the GPU.

The GPU boxes of this build have one B200, so the N > 1 code paths run as
two ranks sharing cuda:0 over the gloo backend (which moves CUDA tensors);
the same calls go over NCCL on an 8-GPU node.  Covered:

* ``encode(grid, cfg, group=...)`` with one expert: every net trains data
  parallel (each rank half of every epoch's batch tiles, one packed gradient
  + loss all-reduce per epoch) -> both ranks hold identical containers whose
  decode matches a single-rank encode's quality;
* ``encode`` with 8 experts: expert parallel (round-robin experts, patches
  per rank, exchange) -> identical to the single-rank container;
* ``decode_full(c, group=...)``: contiguous leaf ranges + gather on rank 0
  -> bit-identical to the single-rank decode;
* ``HybridGrid.query(coords, group=...)``: coordinate slices + gather ->
  bit-identical to the single-rank query;
* the NCCL graph-replayed data-parallel epoch (world-1 NCCL group: capture,
  replay, packed loss pair) -> weights bit-identical to the fused epochs.
"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, backend, fn_name, q):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    kw = {"device_id": torch.device("cuda:0")} if backend == "nccl" else {}
    dist.init_process_group(backend, rank=rank, world_size=world, **kw)
    try:
        q.put((rank, globals()[fn_name](rank, world)))
    except Exception as exc:  # noqa: BLE001
        import traceback
        q.put((rank, RuntimeError(f"rank {rank}: {exc!r}\n{traceback.format_exc()}")))
    finally:
        dist.destroy_process_group()


def _spawn(fn_name, world=2, backend="gloo"):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, backend, fn_name, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    for r, v in out.items():
        if isinstance(v, Exception):
            raise v
    return out


def _weights(c):
    return [np.concatenate([np.asarray(a, np.float32).ravel() for wb in n.params.layers for a in wb])
            for e in sorted(c.experts, key=lambda e: e.id) for _, n in e.nets() if n is not None]


def _small_cfg(**kw):
    from helpers import tiny_cfg
    return tiny_cfg(**kw)


# ---------------------------------------------------------------- data parallel encode

def _dp_encode(rank, world):
    from paper_2208_04448_b200.decoder import decode_full
    from paper_2208_04448_b200.encoder import encode
    from paper_2208_04448_b200.procgen import sphere_sdf
    g = sphere_sdf((31.5, 31.5, 31.5), 24.0, 1.0, 3.0)
    cfg = _small_cfg(max_epochs=40, batch_size=4096, l0_net=(2, 32), voxel_net=(2, 32), ffm_size=32)
    c = encode(g, cfg, device=torch.device("cuda:0"), group=dist.group.WORLD)
    d = decode_full(c, torch.device("cuda:0"))
    iou = _iou(g, d)
    return _weights(c), [n.epochs for e in c.experts for _, n in e.nets() if n is not None], iou


def _iou(truth, got):
    a = {tuple(o): i for i, o in enumerate(truth.leaf_origins)}
    inter = union = 0
    seen = set()
    for j, o in enumerate(got.leaf_origins):
        i = a.get(tuple(o))
        ga = got.leaf_active[j]
        if i is None:
            union += int(ga.sum())
            continue
        seen.add(i)
        ta = truth.leaf_active[i]
        inter += int((ta & ga).sum())
        union += int((ta | ga).sum())
    for i in range(truth.leaf_origins.shape[0]):
        if i not in seen:
            union += int(truth.leaf_active[i].sum())
    return inter / max(union, 1)


def test_data_parallel_encode_two_ranks():
    from paper_2208_04448_b200.decoder import decode_full
    from paper_2208_04448_b200.encoder import encode
    from paper_2208_04448_b200.procgen import sphere_sdf
    out = _spawn("_dp_encode")
    (w0, e0, iou0), (w1, e1, iou1) = out[0], out[1]
    for a, b in zip(w0, w1):
        np.testing.assert_array_equal(a, b)  # identical Adam update on both ranks
    assert e0 == e1
    g = sphere_sdf((31.5, 31.5, 31.5), 24.0, 1.0, 3.0)
    cfg = _small_cfg(max_epochs=40, batch_size=4096, l0_net=(2, 32), voxel_net=(2, 32), ffm_size=32)
    c = encode(g, cfg, device=torch.device("cuda:0"))
    iou1r = _iou(g, decode_full(c, torch.device("cuda:0")))
    print(f"DP encode: IoU {iou0:.5f} (single rank {iou1r:.5f}), epochs {e0}")
    # same sampler stream and update rule; only the cross-rank summation order of
    # the gradient differs from the single-rank fixed order
    assert abs(iou0 - iou1r) < 2e-3
    for a, b in zip(w0, _weights(c)):
        np.testing.assert_allclose(a, b, atol=5e-3)


# ---------------------------------------------------------------- expert parallel encode

def _ep_encode(rank, world):
    from paper_2208_04448_b200.encoder import encode
    from paper_2208_04448_b200.procgen import sphere_sdf
    g = sphere_sdf((512.0, 512.0, 512.0), 30.0, 1.0, 3.0)
    cfg = _small_cfg(max_epochs=30, l0_net=(2, 32), voxel_net=(2, 32), ffm_size=32)
    c = encode(g, cfg, device=torch.device("cuda:0"), group=dist.group.WORLD)
    pats = [(e.id, len(e.patches.l1), len(e.patches.l0)) for e in c.experts]
    return _weights(c), pats


def test_expert_parallel_encode_two_ranks():
    from paper_2208_04448_b200.encoder import encode
    from paper_2208_04448_b200.procgen import sphere_sdf
    out = _spawn("_ep_encode")
    (w0, p0), (w1, p1) = out[0], out[1]
    g = sphere_sdf((512.0, 512.0, 512.0), 30.0, 1.0, 3.0)
    cfg = _small_cfg(max_epochs=30, l0_net=(2, 32), voxel_net=(2, 32), ffm_size=32)
    c = encode(g, cfg, device=torch.device("cuda:0"))
    ref = _weights(c)
    assert len(ref) == len(w0) == len(w1) and len(c.experts) == 8
    # experts are independent: each rank's experts are exactly the single-rank ones
    for a, b, r in zip(w0, w1, ref):
        np.testing.assert_array_equal(a, b)
        np.testing.assert_array_equal(a, r)
    assert p0 == p1 == [(e.id, len(e.patches.l1), len(e.patches.l0)) for e in c.experts]


# ---------------------------------------------------------------- sharded decode / query

def _container():
    from conftest import load_golden
    from paper_2208_04448_b200.model import container_from_arrays
    return container_from_arrays(load_golden("decode_multi"))


def _sharded_decode_full(rank, world):
    from paper_2208_04448_b200.decoder import decode_full
    g = decode_full(_container(), torch.device("cuda:0"), group=dist.group.WORLD)
    if rank != 0:
        assert g is None
        return None
    return g.leaf_origins, g.leaf_active, g.leaf_values, g.l1_child, g.l1_tiles


def test_sharded_decode_full_two_ranks():
    from paper_2208_04448_b200.decoder import decode_full
    out = _spawn("_sharded_decode_full")
    ref = decode_full(_container(), torch.device("cuda:0"))
    got = out[0]
    for a, b in zip(got, (ref.leaf_origins, ref.leaf_active, ref.leaf_values, ref.l1_child, ref.l1_tiles)):
        np.testing.assert_array_equal(a, b)


def _coords():
    rng = np.random.default_rng(5)
    return rng.integers(-40, 300, (200_001, 3)).astype(np.int32)


def _sharded_query(rank, world):
    from paper_2208_04448_b200.decoder import make_hybrid
    h = make_hybrid(_container(), torch.device("cuda:0"))
    v, a = h.query(_coords(), group=dist.group.WORLD)
    return (v, a, h.regressor_evaluations)


def test_sharded_query_two_ranks():
    from paper_2208_04448_b200.decoder import make_hybrid
    out = _spawn("_sharded_query")
    h = make_hybrid(_container(), torch.device("cuda:0"))
    v, a = h.query(_coords())
    np.testing.assert_array_equal(out[0][0].view(np.uint32), v.view(np.uint32))
    np.testing.assert_array_equal(out[0][1], a)
    assert out[1][0] is None
    assert out[0][2] + out[1][2] == h.regressor_evaluations


# ---------------------------------------------------------------- NCCL graph-replayed epochs

def _nccl_graph_epochs(rank, world):
    from helpers import tiny_cfg
    from paper_2208_04448_b200.encoder import DeviceTrainer, init_mlp
    from paper_2208_04448_b200.model import Activation, FourierFeatures
    dev = torch.device("cuda:0")
    rng = np.random.default_rng(12)
    n = 20000
    x = rng.uniform(0, 1, (n, 3)).astype(np.float32)
    y = (0.5 * np.sin(5 * x[:, 0]) * np.cos(3 * x[:, 2])).astype(np.float32)
    ff = FourierFeatures(48, 5.0, 3)
    p0 = init_mlp(96, [64, 64], 1, Activation("sine", 3.0), "linear", 4)
    cfg = tiny_cfg(max_epochs=150, batch_size=4096, lr=1e-3, activation="sine", frequency=3.0)
    fused = DeviceTrainer(p0, ff, x, y, "mse", cfg, 1e-3, 7, True, -1.0, dev)
    fused.run()
    dp = DeviceTrainer(p0, ff, x, y, "mse", cfg, 1e-3, 7, True, -1.0, dev, group=dist.group.WORLD)
    dp.run()
    assert dp._graph is not None  # the epochs after the first were graph replays
    out = []
    for (wa, ba), (wb, bb) in zip(fused.weights().layers, dp.weights().layers):
        out.append((wa, wb, ba, bb))
    lf, ld = fused.status()[2], dp.status()[2]
    res = (out, lf, ld, fused.final(), dp.final())
    fused.close()
    dp.close()
    return res


def test_nccl_graph_replayed_epochs_equal_fused_epochs():
    out = _spawn("_nccl_graph_epochs", world=1, backend="nccl")
    layers, lf, ld, ff, fd = out[0]
    for wa, wb, ba, bb in layers:
        np.testing.assert_array_equal(wa, wb)
        np.testing.assert_array_equal(ba, bb)
    # the loss crosses the all-reduce as an f32 (hi, lo) pair: ~2^-48 relative
    np.testing.assert_allclose(ld, lf, rtol=1e-12)
    assert ff[1] == fd[1] == 150
