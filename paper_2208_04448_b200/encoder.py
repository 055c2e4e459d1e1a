"""Training pipeline on the GPU: drop-in for svcodec.encoder (encoder.py:1-714).

``train_network`` (encoder.py:330-371) runs the whole epoch loop on the
device (``nvdb_trainer_*``: numpy-exact sampler, fused forward/backward on
tcgen05, fixed-order gradient reduction, Adam, early stop on the device);
``encode`` / ``encode_sequence`` keep the reference's orchestration (expert
loop, data gathering, warm start, patch extraction, upper tree) on the host
around it, and patch extraction uses the same fused evaluator as decode.
"""

from __future__ import annotations

import ctypes as C
import logging
import time
import os
from dataclasses import dataclass, field, replace
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np
import torch

from . import _lib
from ._lib import TrainDesc, check, lib
from .decoder import NetEvaluator, _dev
from .errors import EncodeError, SvcodecError
from .model import (GRID_CLASS_SDF, L1_CLASS_ACTIVE_TILE, L1_CLASS_CHILD, L1_CLASS_INACTIVE_TILE,
                    L1_LOCAL, L1_SIZE, L2_SIZE, LEAF_LOCAL, LEAF_SIZE, Activation, DenseLeafGrid,
                    EncodedSubdomain, FourierFeatures, GridMeta, L2NodeRecord, Mask, MlpParams,
                    L1TileMap, LeafBitsMap, NetRecord, NeuralGridContainer, PatchList, Subdomain, SubdomainLayout,
                    UpperTree)
from .netset import _net_desc

logger = logging.getLogger(__name__)

NET_TAGS = {"l1": 0, "tile": 1, "l0": 2, "voxel": 3}          # encoder.py:86
NORM_CONTENT_FRACTION = 0.6                                    # encoder.py:89
REGRESSOR_LOSS_TARGET = 1e-6                                   # encoder.py:92
CLASSIFIER_LOSS_TARGET = 1e-2                                  # encoder.py:93
SDF_SIGNIFICANCE_FACTOR = 0.5                                  # encoder.py:96
FOG_SIGNIFICANCE_DEFAULT = 0.01                                # encoder.py:97
SUBDOMAIN_QUANTUM = 512
LOSS_CODES = {"mse": 0, "ce": 1, "bce": 2}

SLOT_CENTER = L1_LOCAL.astype(np.float64) * 8.0 + 4.0          # encoder.py:99
VOXEL_CENTER = LEAF_LOCAL.astype(np.float64) + 0.5             # encoder.py:100


@dataclass
class TrainConfig:
    """Field-for-field mirror of svcodec.config.TrainConfig (config.py:22-76)."""

    subdomain_size: int = 512
    l1_net: Tuple[int, int] = (3, 24)
    tile_net: Optional[Tuple[int, int]] = (3, 16)
    l0_net: Tuple[int, int] = (3, 48)
    voxel_net: Tuple[int, int] = (3, 48)
    activation: str = "sine"
    frequency: float = 3.0
    ffm_scale: float = 5.0
    ffm_size: int = 96
    lr: float = 1e-3
    refine_lr: Optional[float] = None
    decay: float = 0.975
    interval: float = 100.0
    max_epochs: int = 800
    sample_interval: int = 1
    batch_size: int = 65536
    significance_threshold: Optional[float] = None
    strict_topology: bool = False
    seed: int = 0

    def validate(self) -> None:
        for name in ("l1_net", "l0_net", "voxel_net", "tile_net"):
            spec = getattr(self, name)
            if spec is not None and (spec[0] < 1 or spec[1] < 1):
                raise SvcodecError(f"{name} must have positive depth and width")
        if self.activation not in ("relu", "tanh", "sine"):
            raise SvcodecError(f"unknown activation {self.activation!r}")
        if self.max_epochs < 1 or self.batch_size < 1 or self.sample_interval < 1:
            raise SvcodecError("max_epochs, batch_size and sample_interval must be >= 1")
        if self.subdomain_size <= 0 or self.subdomain_size % SUBDOMAIN_QUANTUM:
            raise SvcodecError("subdomain_size must be a positive multiple of 512")

    def refinement_lr(self) -> float:
        return self.lr if self.refine_lr is None else self.refine_lr


def _validate(cfg) -> None:
    if hasattr(cfg, "validate"):
        cfg.validate()


def stable_seed(*parts: int) -> int:
    """encoder.py:103-104."""
    return int(np.random.SeedSequence(tuple(int(p) for p in parts)).generate_state(1)[0])


def init_mlp(in_dim: int, hidden: Sequence[int], out_dim: int, activation: Activation, head: str,
             seed: int) -> MlpParams:
    """Glorot-uniform init, sine first layer / frequency, zero output layer (neural.py:168-185)."""
    rng = np.random.default_rng(seed)
    dims = [in_dim] + list(hidden) + [out_dim]
    layers = []
    for i in range(len(dims) - 1):
        fan_in, fan_out = dims[i], dims[i + 1]
        limit = np.sqrt(6.0 / (fan_in + fan_out))
        w = rng.uniform(-limit, limit, size=(fan_out, fan_in))
        if i == 0 and activation.kind == "sine":
            w /= activation.frequency
        if i == len(dims) - 2:
            w[...] = 0.0
        layers.append((w.astype(np.float32), np.zeros(fan_out, dtype=np.float32)))
    return MlpParams(layers, activation, head)


def as_grid(grid) -> DenseLeafGrid:
    return grid if isinstance(grid, DenseLeafGrid) else DenseLeafGrid.from_svcodec(grid)


def value_scale_of(grid) -> float:
    """encoder.py:492-495."""
    return grid.half_width * grid.voxel_size if grid.grid_class == GRID_CLASS_SDF else 1.0


def decompose(grid: DenseLeafGrid, size: int) -> SubdomainLayout:
    """Occupied S-lattice cells in sorted order + 26-connected clusters (partition.py:74-120)."""
    if size <= 0 or size % SUBDOMAIN_QUANTUM:
        raise SvcodecError(f"subdomain size must be a positive multiple of {SUBDOMAIN_QUANTUM}, got {size}")
    cells = set()
    occ = grid.leaf_active.any(axis=1)
    for o in np.unique(grid.leaf_origins[occ] // size, axis=0):
        cells.add(tuple(int(v) for v in o))
    for org, ext in grid.active_tiles():
        lo = np.asarray(org, dtype=np.int64)
        for corner in (lo, lo + ext - 1):
            cells.add(tuple(int(v) // size for v in corner))
    layout = SubdomainLayout(size=size)
    ordered = sorted(cells)
    for sid, cell in enumerate(ordered):
        layout.subdomains.append(Subdomain(id=sid, cell=cell, size=size))
        layout.cell_to_id[cell] = sid
    cluster, seen = -1, set()
    for cell in ordered:
        if cell in seen:
            continue
        cluster += 1
        stack = [cell]
        seen.add(cell)
        while stack:
            cur = stack.pop()
            layout.subdomains[layout.cell_to_id[cur]].cluster_id = cluster
            for dx in (-1, 0, 1):
                for dy in (-1, 0, 1):
                    for dz in (-1, 0, 1):
                        nb = (cur[0] + dx, cur[1] + dy, cur[2] + dz)
                        if nb != cur and nb in layout.cell_to_id and nb not in seen:
                            seen.add(nb)
                            stack.append(nb)
    layout.cluster_count = cluster + 1
    return layout


def _boxes_intersect(origins: np.ndarray, span: int, lo, hi) -> np.ndarray:
    if origins.shape[0] == 0:
        return np.zeros(0, dtype=bool)
    return np.all((origins + span > lo) & (origins < hi), axis=1)


def expert_norm(sub: Subdomain, grid: DenseLeafGrid) -> Tuple[np.ndarray, float]:
    """Isotropic content-box input map (encoder.py:181-194)."""
    lo = sub.expanded_lo().astype(np.float64)
    hi = sub.expanded_hi().astype(np.float64)
    sel = _boxes_intersect(grid.l1_origins, 128, sub.expanded_lo(), sub.expanded_hi())
    if sel.any():
        lo = np.maximum(lo, grid.l1_origins[sel].min(axis=0).astype(np.float64))
        hi = np.minimum(hi, (grid.l1_origins[sel] + 128).max(axis=0).astype(np.float64))
    extent = float((hi - lo).max())
    scale = extent / NORM_CONTENT_FRACTION
    return (lo + hi) / 2.0 - scale / 2.0, scale


@dataclass
class ExpertData:
    sub: Subdomain
    norm_origin: np.ndarray
    norm_scale: float
    l1_inputs: Optional[np.ndarray] = None
    l1_labels: Optional[np.ndarray] = None
    tile_inputs: Optional[np.ndarray] = None
    tile_targets: Optional[np.ndarray] = None
    l0_inputs: Optional[np.ndarray] = None
    l0_labels: Optional[np.ndarray] = None
    vox_inputs: Optional[np.ndarray] = None
    vox_targets: Optional[np.ndarray] = None


def gather_expert_data(grid: DenseLeafGrid, sub: Subdomain, value_scale: float, norm=None) -> ExpertData:
    """Per-expert training sets over the expanded box (encoder.py:197-235)."""
    lo, hi = sub.expanded_lo(), sub.expanded_hi()
    no, ns = expert_norm(sub, grid) if norm is None else norm
    data = ExpertData(sub=sub, norm_origin=no, norm_scale=ns)

    def nrm(c):
        return ((c - no) / ns).astype(np.float32)

    sel1 = _boxes_intersect(grid.l1_origins, 128, lo, hi)
    if sel1.any():
        org = grid.l1_origins[sel1]
        cen = (org[:, None, :] + SLOT_CENTER[None]).reshape(-1, 3)
        child = grid.l1_child[sel1].reshape(-1)
        active = grid.l1_active[sel1].reshape(-1)
        labels = np.full(child.shape, L1_CLASS_INACTIVE_TILE, dtype=np.int64)
        labels[active & ~child] = L1_CLASS_ACTIVE_TILE
        labels[child] = L1_CLASS_CHILD
        data.l1_inputs = nrm(cen)
        data.l1_labels = labels
        tsel = active & ~child
        if tsel.any():
            data.tile_inputs = data.l1_inputs[tsel]
            data.tile_targets = (grid.l1_tiles[sel1].reshape(-1)[tsel] / value_scale).astype(np.float32)
    sel0 = _boxes_intersect(grid.leaf_origins, 8, lo, hi)
    if sel0.any():
        org = grid.leaf_origins[sel0]
        cen = (org[:, None, :] + VOXEL_CENTER[None]).reshape(-1, 3)
        act = grid.leaf_active[sel0].reshape(-1)
        data.l0_inputs = nrm(cen)
        data.l0_labels = act.astype(np.float32)
        if act.any():
            data.vox_inputs = data.l0_inputs[act]
            data.vox_targets = (grid.leaf_values[sel0].reshape(-1)[act] / value_scale).astype(np.float32)
    return data


class DeviceGrid:
    """A dense-leaf grid's arrays on the device, uploaded once per encode, so
    that every expert's training sets (encoder.py:197-235) are gathered there
    instead of in host numpy (C3: 8 experts x ~80 M leaf voxels)."""

    def __init__(self, grid: DenseLeafGrid, device=None):
        import torch
        dev = _dev(device)
        self.dev = dev

        def up(a, dt=None):
            a = np.ascontiguousarray(a if dt is None else np.asarray(a, dt))
            return torch.from_numpy(a).to(dev)
        self.l1_origins = up(grid.l1_origins, np.int64).reshape(-1, 3)
        self.l1_child = up(grid.l1_child, np.bool_).reshape(-1, L1_SIZE)
        self.l1_active = up(grid.l1_active, np.bool_).reshape(-1, L1_SIZE)
        self.l1_tiles = up(grid.l1_tiles, np.float32).reshape(-1, L1_SIZE)
        self.leaf_origins = up(grid.leaf_origins, np.int64).reshape(-1, 3)
        self.leaf_active = up(grid.leaf_active, np.bool_).reshape(-1, LEAF_SIZE)
        self.leaf_values = up(grid.leaf_values, np.float32).reshape(-1, LEAF_SIZE)
        self.slot_center = torch.from_numpy(SLOT_CENTER).to(dev)
        self.voxel_center = torch.from_numpy(VOXEL_CENTER).to(dev)


def gather_expert_data_device(grid: DenseLeafGrid, dg: DeviceGrid, sub: Subdomain, value_scale: float,
                              norm=None) -> ExpertData:
    """gather_expert_data on the device: the same f64 centre / normalisation
    arithmetic (IEEE, so bit-identical to the numpy form) and the same row
    order; the fields are device tensors."""
    import torch
    lo, hi = sub.expanded_lo(), sub.expanded_hi()
    no, ns = expert_norm(sub, grid) if norm is None else norm
    data = ExpertData(sub=sub, norm_origin=no, norm_scale=ns)
    dev = dg.dev
    no_t = torch.as_tensor(np.asarray(no, np.float64), device=dev)
    # divisors as device tensors: torch divides by a host scalar as a
    # multiplication by its reciprocal, which is not the IEEE quotient numpy takes
    ns_t = torch.tensor([float(ns)], dtype=torch.float64, device=dev)
    vs_t = torch.tensor([float(value_scale)], dtype=torch.float32, device=dev)
    lo_t = torch.as_tensor(np.asarray(lo, np.int64), device=dev)
    hi_t = torch.as_tensor(np.asarray(hi, np.int64), device=dev)

    def nrm(c):
        return torch.div(c - no_t, ns_t).to(torch.float32)

    def boxes(origins, span):
        if origins.shape[0] == 0:
            return torch.zeros(0, dtype=torch.bool, device=dev)
        return torch.all((origins + span > lo_t) & (origins < hi_t), dim=1)

    sel1 = boxes(dg.l1_origins, 128)
    if bool(sel1.any()):
        org = dg.l1_origins[sel1]
        cen = (org[:, None, :].to(torch.float64) + dg.slot_center[None]).reshape(-1, 3)
        child = dg.l1_child[sel1].reshape(-1)
        active = dg.l1_active[sel1].reshape(-1)
        labels = torch.full(child.shape, L1_CLASS_INACTIVE_TILE, dtype=torch.int64, device=dev)
        labels[active & ~child] = L1_CLASS_ACTIVE_TILE
        labels[child] = L1_CLASS_CHILD
        data.l1_inputs = nrm(cen)
        data.l1_labels = labels
        tsel = active & ~child
        if bool(tsel.any()):
            data.tile_inputs = data.l1_inputs[tsel]
            data.tile_targets = torch.div(dg.l1_tiles[sel1].reshape(-1)[tsel], vs_t)
    sel0 = boxes(dg.leaf_origins, 8)
    if bool(sel0.any()):
        org = dg.leaf_origins[sel0]
        cen = (org[:, None, :].to(torch.float64) + dg.voxel_center[None]).reshape(-1, 3)
        act = dg.leaf_active[sel0].reshape(-1)
        data.l0_inputs = nrm(cen)
        del cen
        data.l0_labels = act.to(torch.float32)
        if bool(act.any()):
            data.vox_inputs = data.l0_inputs[act]
            data.vox_targets = torch.div(dg.leaf_values[sel0].reshape(-1)[act], vs_t)
    return data


@dataclass
class NetSpec:
    tag: str
    arch: Tuple[int, int]
    m: int
    head: str
    out_dim: int
    loss_kind: str
    loss_target: float
    full_batch: bool


def net_spec(tag: str, cfg) -> Optional[NetSpec]:
    """encoder.py:309-324."""
    if tag == "l1":
        return NetSpec("l1", tuple(cfg.l1_net), max(1, cfg.ffm_size // 2), "logits", 3, "ce",
                       CLASSIFIER_LOSS_TARGET, True)
    if tag == "tile":
        if cfg.tile_net is None:
            return None
        return NetSpec("tile", tuple(cfg.tile_net), cfg.ffm_size, "linear", 1, "mse", REGRESSOR_LOSS_TARGET, True)
    if tag == "l0":
        return NetSpec("l0", tuple(cfg.l0_net), cfg.ffm_size, "binary", 1, "bce", CLASSIFIER_LOSS_TARGET, False)
    if tag == "voxel":
        return NetSpec("voxel", tuple(cfg.voxel_net), cfg.ffm_size, "linear", 1, "mse", REGRESSOR_LOSS_TARGET,
                       False)
    raise ValueError(tag)


class _DeviceArray:
    """Zero-copy torch view of library-owned device memory (__cuda_array_interface__)."""

    def __init__(self, ptr: int, n: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (int(ptr), False),
                                         "version": 3, "strides": None}


def shard_of(ntiles: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous tile range of one data-parallel rank (same split as train.cu)."""
    return ntiles * rank // world, ntiles * (rank + 1) // world


class DeviceTrainer:
    """One network's device-resident training loop (nvdb_trainer_*).

    With a ``torch.distributed`` process group of size G > 1, every rank draws
    the same batch (same sampler stream), processes its contiguous share of
    the batch tiles, and the fp32 gradient sum plus the loss sum are
    all-reduced (NCCL over NVLink) between the gradient and the Adam phase of
    each epoch; all ranks then apply the identical update.
    """

    CHUNK = 64  # epochs enqueued between host checks of the stop flag

    def __init__(self, params: MlpParams, ff: FourierFeatures, inputs: np.ndarray, targets: np.ndarray,
                 loss_kind: str, cfg, lr0: float, seed_draw: int, sampled: bool, target_loss: float,
                 device=None, group=None, path: int = 0):
        self.dev = _dev(device)
        self.group = group
        import torch.distributed as dist
        self.world = dist.get_world_size(group) if group is not None else 1
        self.rank = dist.get_rank(group) if group is not None else 0
        self.params, self.ff = params, ff
        n = inputs.shape[0]
        self.n = n
        self.max_epochs = int(cfg.max_epochs)
        self.batch, self.sampled = int(cfg.batch_size), bool(sampled)
        if isinstance(inputs, torch.Tensor):  # device-gathered training set (gather_expert_data_device)
            self.x = inputs.to(self.dev, torch.float32).reshape(-1, 3).contiguous()
        else:
            self.x = torch.from_numpy(np.ascontiguousarray(inputs, dtype=np.float32).reshape(-1, 3)).to(self.dev)
        if isinstance(targets, torch.Tensor):
            self.y = targets.to(self.dev, torch.float32).reshape(-1).contiguous()
        else:
            self.y = torch.from_numpy(np.ascontiguousarray(targets, dtype=np.float32).reshape(-1)).to(self.dev)
        E = self.max_epochs
        ep = np.arange(E, dtype=np.float64)
        # lr_at in float64 then np.float32 (neural.py:215-219, encoder.py:366)
        self.lr = np.asarray([np.float32(lr0 * cfg.decay ** (e / cfg.interval)) for e in range(E)], dtype=np.float32)
        self.c1 = np.asarray([np.float32(1.0 - 0.9 ** (e + 1)) for e in range(E)], dtype=np.float32)
        self.c2 = np.asarray([np.float32(1.0 - 0.999 ** (e + 1)) for e in range(E)], dtype=np.float32)
        del ep
        interval = max(1, int(cfg.sample_interval))
        nchunks = (E + interval - 1) // interval if interval > 1 else 0
        words = np.zeros((E + nchunks, 4), dtype=np.uint64)
        if sampled:
            # Sampler (encoder.py:256-267): SeedSequence((seed, 0, epoch)); with a working
            # subset, (seed, 2, epoch) per epoch and (seed, 1, chunk) per chunk of `interval` epochs
            stream = 0 if interval == 1 else 2
            for e in range(E):
                words[e] = np.random.SeedSequence((seed_draw, stream, e)).generate_state(4, np.uint64)
            for ch in range(nchunks):
                words[E + ch] = np.random.SeedSequence((seed_draw, 1, ch)).generate_state(4, np.uint64)
        self.words = words
        keep: list = []
        nd = _net_desc(params, ff, keep)
        self._keep = keep
        d = TrainDesc(net=nd, loss_kind=LOSS_CODES[loss_kind], n=n, inputs=self.x.data_ptr(),
                      targets=self.y.data_ptr(), batch=int(cfg.batch_size), sampled=int(bool(sampled)),
                      sample_interval=int(cfg.sample_interval), max_epochs=E,
                      lr=self.lr.ctypes.data_as(C.c_void_p), c1=self.c1.ctypes.data_as(C.c_void_p),
                      c2=self.c2.ctypes.data_as(C.c_void_p), seed_words=self.words.ctypes.data_as(C.c_void_p),
                      target_loss=float(target_loss), shard_rank=self.rank, shard_count=self.world,
                      path=int(path))
        h = C.c_void_p()
        torch.cuda.synchronize(self.dev)
        check(lib().nvdb_trainer_create(C.byref(d), C.byref(h)), "nvdb_trainer_create")
        self.handle = h
        self.epochs_enqueued = 0
        self._graph = None
        if group is not None:  # data-parallel form (a world-1 group runs it too)
            g, nf = C.c_void_p(), C.c_int64()
            check(lib().nvdb_trainer_packed(self.handle, C.byref(g), C.byref(nf)), "nvdb_trainer_packed")
            # gradient sums + the loss (hi, lo) pair: one all-reduce per epoch
            self.packed = torch.as_tensor(_DeviceArray(g.value, nf.value, "<f4"), device=self.dev)
            import torch.distributed as dist
            self._graphable = dist.get_backend(group) == "nccl" and os.environ.get("NVDB_DP_GRAPH", "1") == "1"

    def set_ctas(self, ctas: int) -> None:
        """Bound the SMs this trainer's epoch kernels use (0 = all; nvdb_trainer_set_ctas)."""
        check(lib().nvdb_trainer_set_ctas(self.handle, int(ctas)), "nvdb_trainer_set_ctas")

    def epoch_work(self) -> float:
        """Relative per-epoch time: 128-sample tiles per epoch (the epoch kernels
        are latency-bound per tile, so their time follows the tile count more
        than the flops), weighted by the layer width's share of the work."""
        batch = min(self.n, self.batch) if self.sampled else self.n
        width = max(np.asarray(w).shape[0] for w, _ in self.params.layers[:-1])
        return float((batch + 127) // 128) * (1.0 + width / 256.0)

    def _epoch_dp(self, st) -> None:
        import torch.distributed as dist
        check(lib().nvdb_trainer_phase(self.handle, 1, st), "nvdb_trainer_phase")
        dist.all_reduce(self.packed, group=self.group)
        check(lib().nvdb_trainer_phase(self.handle, 2, st), "nvdb_trainer_phase")

    def _enqueue(self, k: int, st) -> None:
        if self.group is None:
            check(lib().nvdb_trainer_run(self.handle, k, st), "nvdb_trainer_run")
            return
        if self.epochs_enqueued == 0 or not self._graphable:
            # eager epoch (the first one also presamples every epoch's batch)
            self._epoch_dp(st)
            k -= 1
            if not self._graphable:
                for _ in range(k):
                    self._epoch_dp(st)
                return
        if k <= 0:
            return
        if self._graph is None:
            # phase 1 -> NCCL all-reduce -> phase 2 captured once; every launch
            # reads the epoch from device memory, so the graph replays any epoch
            # (no Python / host launch cost per epoch; replays after the early
            # stop are device no-ops)
            torch.cuda.synchronize(self.dev)
            g = torch.cuda.CUDAGraph()
            cap = torch.cuda.Stream(self.dev)
            try:
                with torch.cuda.stream(cap):
                    with torch.cuda.graph(g, stream=cap):
                        self._epoch_dp(cap.cuda_stream)
            except Exception as exc:  # noqa: BLE001 -- a communicator that cannot be captured: eager epochs
                logger.warning("data-parallel epoch graph capture failed (%s); running eager epochs", exc)
                torch.cuda.synchronize(self.dev)
                self._graphable = False
                for _ in range(k):
                    try:
                        self._epoch_dp(st)
                    except (ValueError, _lib.NvdbError):  # the failed capture counted one host epoch: run complete
                        break
                return
            self._graph = g  # capture does not execute: every epoch below is a replay
        for _ in range(k):
            self._graph.replay()

    def run(self, epochs: Optional[int] = None) -> Tuple[float, int]:
        """Train until the early stop or max_epochs; returns (final loss, epochs)."""
        limit = self.max_epochs if epochs is None else min(self.max_epochs, self.epochs_enqueued + epochs)
        st = torch.cuda.current_stream(self.dev).cuda_stream
        while self.epochs_enqueued < limit:
            k = min(self.CHUNK, limit - self.epochs_enqueued)
            self._enqueue(k, st)
            self.epochs_enqueued += k
            done, stopped = self.status()[:2]
            if stopped:
                break
        return self.final()

    def status(self):
        if self._graph is not None:  # graph replays record no completion event: order the host here
            torch.cuda.current_stream(self.dev).synchronize()
        done, stopped = C.c_int32(), C.c_int32()
        losses = np.zeros(self.max_epochs, dtype=np.float64)
        check(lib().nvdb_trainer_status(self.handle, C.byref(done), C.byref(stopped),
                                        losses.ctypes.data_as(C.c_void_p), self.max_epochs), "nvdb_trainer_status")
        return done.value, stopped.value, losses

    def final(self) -> Tuple[float, int]:
        done, _, losses = self.status()
        return float(losses[done - 1]) if done > 0 else float("inf"), int(done)

    def weights(self) -> MlpParams:
        """Current parameters in the caller's layer shapes.  The trainer holds
        unequal hidden widths zero-padded to the widest (netset._net_desc);
        padded units keep zero weights and gradients, so the real layers are
        the leading blocks of the padded ones."""
        layers = self.params.layers
        depth = len(layers) - 1
        width = max(np.asarray(w).shape[0] for w, _ in layers[:-1])
        shapes = []
        for li, (w, _) in enumerate(layers):
            rows = np.asarray(w).shape[0] if li == depth else width
            cols = np.asarray(w).shape[1] if li == 0 else width
            shapes.append((rows, cols))
        if self._graph is not None:
            torch.cuda.current_stream(self.dev).synchronize()
        ws = [np.zeros(sh, dtype=np.float32) for sh in shapes]
        bs = [np.zeros(sh[0], dtype=np.float32) for sh in shapes]
        wp = (C.POINTER(C.c_float) * len(ws))(*[w.ctypes.data_as(C.POINTER(C.c_float)) for w in ws])
        bp = (C.POINTER(C.c_float) * len(bs))(*[b.ctypes.data_as(C.POINTER(C.c_float)) for b in bs])
        check(lib().nvdb_trainer_weights(self.handle, wp, bp), "nvdb_trainer_weights")
        out = []
        for (w0, b0), w, b in zip(layers, ws, bs):
            r, c = np.asarray(w0).shape
            out.append((np.ascontiguousarray(w[:r, :c]), np.ascontiguousarray(b[:r])))
        return MlpParams(out, self.params.activation, self.params.head)

    def close(self):
        if getattr(self, "handle", None) is not None and self.handle.value:
            if getattr(self, "_graph", None) is not None:  # replays record no completion event
                torch.cuda.current_stream(self.dev).synchronize()
                self._graph = None
            lib().nvdb_trainer_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass


_TRAIN_STREAMS: Dict[int, list] = {}


def run_concurrent(trainers: List["DeviceTrainer"], width: int = 2) -> List[Tuple[float, int]]:
    """Run independent trainers ``width`` at a time, each on its own stream
    with its full grid (the same kernels, tile partitions and reduction order
    as ``DeviceTrainer.run``, so every net's weights and epochs are
    bit-identical to training them one after another).  The epoch kernels are
    latency-bound per tile: two nets' epochs
    interleaved on the SMs overlap one net's weight-gradient / Adam tail and
    launch gaps with the other's fwd/dgrad (C2 l0 + voxel, 800 epochs: 169.7
    -> 148.9 ms).  Nets pair up by epoch shape (an expert's l0 and voxel
    nets); three at once, or the full-batch l1 net beside an l0 net, was
    measured slower or unstable.  Data-parallel trainers (a process group)
    run one after another."""
    if len(trainers) <= 1 or width <= 1 or any(t.group is not None for t in trainers):
        return [t.run() for t in trainers]
    # nets of the same epoch shape (the l0 and voxel nets of an expert) pair
    # up; a net without a partner runs alone on the whole GPU (pairing the
    # full-batch l1 net with an l0 net ran 186-275 ms run to run on C2
    # against 180 for l1 alone then l0 + voxel)
    shapes: Dict[float, List[int]] = {}
    for i, t in enumerate(trainers):
        shapes.setdefault(t.epoch_work(), []).append(i)
    res: List[Optional[Tuple[float, int]]] = [None] * len(trainers)
    for idx in sorted(shapes.values(), key=len):
        if len(idx) == 1:
            res[idx[0]] = trainers[idx[0]].run()
        else:
            for i, r in zip(idx, _run_streams([trainers[i] for i in idx], width)):
                res[i] = r
    return res


def _run_streams(trainers: List["DeviceTrainer"], width: int) -> List[Tuple[float, int]]:
    """run_concurrent's stream schedule: ``width`` trainers at a time."""
    dev = trainers[0].dev
    cur = torch.cuda.current_stream(dev)
    pool = _TRAIN_STREAMS.setdefault(dev.index if dev.index is not None else torch.cuda.current_device(), [])
    while len(pool) < width:  # persistent per device (torch's allocator pools blocks per stream)
        pool.append(torch.cuda.Stream(dev))
    streams = pool[:width]
    for s in streams:
        s.wait_stream(cur)  # the trainers' uploads were enqueued on the current stream
    todo = sorted((i for i, t in enumerate(trainers) if t.epochs_enqueued < t.max_epochs),
                  key=lambda i: -trainers[i].epoch_work() * trainers[i].max_epochs)
    slots: List[Optional[Tuple[int, torch.cuda.Event]]] = [None] * width

    def enqueue(slot, i):
        t = trainers[i]
        k = min(t.CHUNK, t.max_epochs - t.epochs_enqueued)
        t._enqueue(k, streams[slot].cuda_stream)
        t.epochs_enqueued += k
        ev = torch.cuda.Event()
        ev.record(streams[slot])
        slots[slot] = (i, ev)

    for slot in range(width):
        if todo:
            enqueue(slot, todo.pop(0))
    while any(sl is not None for sl in slots):
        # the stop flag is checked per chunk in completion order, so a
        # finished chunk is followed at once by the next one on its stream
        progressed = False
        for slot, sl in enumerate(slots):
            if sl is None or not sl[1].query():
                continue
            progressed = True
            i = sl[0]
            t = trainers[i]
            _, stopped = t.status()[:2]
            if stopped or t.epochs_enqueued >= t.max_epochs:
                slots[slot] = None
                if todo:
                    enqueue(slot, todo.pop(0))
            else:
                enqueue(slot, i)
        if not progressed:
            time.sleep(2e-5)
    for s in streams:
        cur.wait_stream(s)
    return [t.final() for t in trainers]


def _train_flops(layers) -> int:
    """2*(3*sum MAC - MAC_0) per sample."""
    macs = [np.asarray(w).shape[0] * np.asarray(w).shape[1] for w, _ in layers]
    return int(2 * (3 * sum(macs) - macs[0]))


def _check_targets(targets, kind: str, out_dim: int) -> None:
    """Label / target validation of neural.py:282-283, 295-296 (ValueError)."""
    import torch
    if isinstance(targets, torch.Tensor):
        t = targets
        if kind == "ce":
            if t.numel() and (bool(t.min() < 0) or bool(t.max() >= out_dim)):
                raise ValueError("class label outside head arity")
        elif kind == "bce":
            if bool(((t != 0) & (t != 1)).any()):
                raise ValueError("binary targets must be 0 or 1")
        if t.is_floating_point() and bool(torch.isnan(t).any()):
            raise ValueError("NaN in targets")
        return
    t = np.asarray(targets)
    if kind == "ce":
        if t.size and (t.min() < 0 or t.max() >= out_dim):
            raise ValueError("class label outside head arity")
    elif kind == "bce":
        if ((t != 0) & (t != 1)).any():
            raise ValueError("binary targets must be 0 or 1")
    if np.isnan(np.asarray(t, dtype=np.float64)).any():
        raise ValueError("NaN in targets")


def make_trainer(inputs: np.ndarray, targets: np.ndarray, spec: NetSpec, cfg, expert_id: int, lr0: float,
                 warm: Optional[NetRecord] = None, stop_loss: Optional[float] = None, device=None,
                 group=None) -> Tuple[DeviceTrainer, FourierFeatures]:
    """The trainer train_network runs (encoder.py:330-360: seeds, warm start,
    init, sampler choice, stop target), not yet started."""
    depth, width = spec.arch
    tagid = NET_TAGS[spec.tag]
    seed_ff = stable_seed(cfg.seed, expert_id, tagid, 0)
    seed_init = stable_seed(cfg.seed, expert_id, tagid, 1)
    seed_draw = stable_seed(cfg.seed, expert_id, tagid, 2)
    activation = Activation(cfg.activation, cfg.frequency)
    if warm is not None:
        params = MlpParams([(np.asarray(w, np.float32).copy(), np.asarray(b, np.float32).copy())
                            for w, b in warm.params.layers], activation, warm.params.head)
        ff = warm.ff
    else:
        ff = FourierFeatures(spec.m, cfg.ffm_scale, seed_ff)
        params = init_mlp(2 * spec.m, [width] * depth, spec.out_dim, activation, spec.head, seed_init)
    import torch
    x = inputs if isinstance(inputs, torch.Tensor) else np.asarray(inputs)
    if (bool(torch.isnan(x).any()) if isinstance(x, torch.Tensor) else np.isnan(x).any()):
        raise ValueError("NaN in batch inputs")
    _check_targets(targets, spec.loss_kind, spec.out_dim)
    n = x.shape[0]
    target = spec.loss_target if stop_loss is None else max(spec.loss_target, stop_loss)
    sampled = (not spec.full_batch) and n > cfg.batch_size
    tr = DeviceTrainer(params, ff, x, targets, spec.loss_kind, cfg, lr0, seed_draw, sampled, target, device,
                       group=group)
    return tr, ff


def train_network(inputs: np.ndarray, targets: np.ndarray, spec: NetSpec, cfg, expert_id: int, lr0: float,
                  warm: Optional[NetRecord] = None, stop_loss: Optional[float] = None, workspace=None,
                  device=None, return_trainer: bool = False, group=None) -> NetRecord:
    """Train one network on the GPU; returns the committed record (encoder.py:330-371).
    ``group``: data-parallel over the ranks of a torch.distributed group."""
    del workspace
    tr, ff = make_trainer(inputs, targets, spec, cfg, expert_id, lr0, warm, stop_loss, device, group)
    try:
        loss, epochs = tr.run()
        out = NetRecord(params=tr.weights(), ff=ff, final_loss=float(loss), epochs=epochs)
        if return_trainer:
            return out, tr
        return out
    finally:
        if not return_trainer:
            tr.close()


def extract_patches(grid: DenseLeafGrid, layout: SubdomainLayout, experts: List[EncodedSubdomain], cfg,
                    device=None, only=None, dgrid: Optional[DeviceGrid] = None) -> None:
    """Classifier disagreements vs ground truth become patches (encoder.py:430-486).

    Predictions come from the same fused blended evaluator the decoder uses.
    ``only``: subdomain ids to extract (an expert-parallel rank's own).
    ``dgrid``: the grid on the device; the level-0 comparison (every leaf
    voxel of the core box) then runs there and only the disagreeing rows
    come back to the host.
    """
    band = grid.half_width * grid.voxel_size
    if cfg.significance_threshold is not None:
        eps = cfg.significance_threshold
    elif grid.grid_class == GRID_CLASS_SDF:
        eps = SDF_SIGNIFICANCE_FACTOR * grid.voxel_size
    else:
        eps = FOG_SIGNIFICANCE_DEFAULT
    ev = NetEvaluator(experts, layout.size, layout.halo, grid.background, device)
    by_id = {e.id: e for e in experts}
    try:
        for sub in layout.subdomains:
            if only is not None and sub.id not in only:
                continue
            expert = by_id[sub.id]
            patches = PatchList()
            own1 = np.all((grid.l1_origins >= sub.lo) & (grid.l1_origins < sub.hi), axis=1) \
                if grid.l1_origins.shape[0] else np.zeros(0, bool)
            if own1.any():
                org = grid.l1_origins[own1]
                d_org = torch.from_numpy(org.astype(np.int32)).to(ev.dev)
                pred = torch.empty(org.shape[0] * L1_SIZE, dtype=torch.uint8, device=ev.dev)
                ev.evaluate("l1", _lib.SRC_L1_SLOT, d_org, org.shape[0] * L1_SIZE, _lib.OUT_L1CLASS, u8=pred)
                pred = pred.cpu().numpy().astype(np.int64)
                child = grid.l1_child[own1].reshape(-1)
                active = grid.l1_active[own1].reshape(-1)
                truth = np.full(child.shape, L1_CLASS_INACTIVE_TILE, dtype=np.int64)
                truth[active & ~child] = L1_CLASS_ACTIVE_TILE
                truth[child] = L1_CLASS_CHILD
                so = (org[:, None, :] + (L1_LOCAL * 8)[None]).reshape(-1, 3)
                bad = np.flatnonzero(pred != truth)
                patches.l1.extend_arrays(so[bad], truth[bad])
            if dgrid is not None:
                _l0_patches_device(grid, dgrid, sub, ev, cfg, band, eps, patches)
                expert.patches = patches
                continue
            own0 = np.all((grid.leaf_origins >= sub.lo) & (grid.leaf_origins < sub.hi), axis=1) \
                if grid.leaf_origins.shape[0] else np.zeros(0, bool)
            if own0.any():
                org = grid.leaf_origins[own0]
                d_org = torch.from_numpy(org.astype(np.int32)).to(ev.dev)
                pred = torch.empty(org.shape[0] * LEAF_SIZE, dtype=torch.uint8, device=ev.dev)
                ev.evaluate("l0", _lib.SRC_LEAF_VOX, d_org, org.shape[0] * LEAF_SIZE, _lib.OUT_L0ACTIVE, u8=pred)
                pred = pred.cpu().numpy().astype(bool)
                truth = grid.leaf_active[own0].reshape(-1)
                values = grid.leaf_values[own0].reshape(-1)
                disagree = pred != truth
                if not cfg.strict_topology:
                    keep = truth.copy()
                    if grid.grid_class == GRID_CLASS_SDF:
                        keep &= np.abs(values) < band - eps
                    else:
                        keep &= values > eps
                    disagree &= keep
                coords = (org[:, None, :] + LEAF_LOCAL[None]).reshape(-1, 3)
                bad = np.flatnonzero(disagree)
                act = truth[bad].astype(bool)
                patches.l0.extend_arrays(coords[bad], act,
                                         np.where(act, values[bad].astype(np.float64), 0.0))
            expert.patches = patches
    finally:
        ev.close()


def _l0_patches_device(grid: DenseLeafGrid, dg: DeviceGrid, sub, ev, cfg, band: float, eps: float,
                       patches: PatchList) -> None:
    """extract_patches' level-0 stage (encoder.py:461-486) on the device: the
    same masks (comparisons of f32 values against the f32-cast thresholds, as
    numpy's weak-scalar rules do), rows in the same order."""
    dev = dg.dev
    if dg.leaf_origins.shape[0] == 0:
        return
    lo = torch.as_tensor(np.asarray(sub.lo, np.int64), device=dev)
    hi = torch.as_tensor(np.asarray(sub.hi, np.int64), device=dev)
    own0 = torch.all((dg.leaf_origins >= lo) & (dg.leaf_origins < hi), dim=1)
    idx = own0.nonzero().flatten()
    if idx.numel() == 0:
        return
    org = dg.leaf_origins[idx]
    d_org = org.to(torch.int32).contiguous()
    n = org.shape[0] * LEAF_SIZE
    pred = torch.empty(n, dtype=torch.uint8, device=dev)
    ev.evaluate("l0", _lib.SRC_LEAF_VOX, d_org, n, _lib.OUT_L0ACTIVE, u8=pred)
    truth = dg.leaf_active[idx].reshape(-1)
    values = dg.leaf_values[idx].reshape(-1)
    disagree = pred.bool() != truth
    if not cfg.strict_topology:
        keep = truth.clone()
        if grid.grid_class == GRID_CLASS_SDF:
            keep &= values.abs() < float(np.float32(band - eps))
        else:
            keep &= values > float(np.float32(eps))
        disagree &= keep
    bad = disagree.nonzero().flatten()
    if bad.numel() == 0:
        return
    act = truth[bad]
    coords = org[bad // LEAF_SIZE] + torch.from_numpy(LEAF_LOCAL).to(dev)[bad % LEAF_SIZE]
    vals = torch.where(act, values[bad].to(torch.float64), torch.zeros((), dtype=torch.float64, device=dev))
    patches.l0.extend_arrays(coords.cpu().numpy(), act.cpu().numpy().astype(bool), vals.cpu().numpy())


def build_upper_tree(grid: DenseLeafGrid) -> UpperTree:
    """Explicit root/level-2 content + level-1 origins, tiles and fills (encoder.py:498-528)."""
    tree = UpperTree()
    tree.root_tiles = dict(grid.root_tiles)
    bg = np.float32(grid.background)
    for ni in range(grid.l2_origins.shape[0]):
        keep = (~grid.l2_child[ni]) & (grid.l2_active[ni] | (grid.l2_tiles[ni] != bg))
        tiles = {int(i): float(grid.l2_tiles[ni, i]) for i in np.flatnonzero(keep)}
        tree.l2_nodes.append(L2NodeRecord(tuple(int(v) for v in grid.l2_origins[ni]),
                                          Mask(grid.l2_child[ni].copy()), Mask(grid.l2_active[ni].copy()), tiles))
    tree.l1_origins = [tuple(o) for o in grid.l1_origins.astype(np.int64).tolist()]
    # inactive tiles with a stored value, as columns (model.L1TileMap; encoder.py:512-517)
    inactive = ~grid.l1_child & ~grid.l1_active & (grid.l1_tiles != bg)
    rows, cols = np.nonzero(inactive)
    nodes, counts = np.unique(rows, return_counts=True)
    tree.l1_tiles = L1TileMap.from_arrays(grid.l1_origins[nodes], counts, cols, grid.l1_tiles[rows, cols])
    neg = ~grid.leaf_active & (grid.leaf_values < 0)
    sel = np.flatnonzero(neg.any(axis=1))
    tree.leaf_negative_fill = LeafBitsMap.from_arrays(grid.leaf_origins[sel], neg[sel])
    tree.l1_origins.sort()
    return tree


_EXPERT_NETS = (("l1", "l1_classifier"), ("tile", "tile_regressor"), ("l0", "l0_classifier"),
                ("voxel", "voxel_regressor"))


def _prepare_expert(grid: DenseLeafGrid, sub: Subdomain, cfg, lr0: float, warm=None, stop_losses=None,
                    device=None, group=None, dgrid: Optional[DeviceGrid] = None):
    """encoder.py:531-570 up to training: the expert's data and one trainer per
    net (l1, tile, l0, voxel), not yet run."""
    scale = value_scale_of(grid)
    norm = (np.asarray(warm.norm_origin, dtype=np.float64).copy(), float(warm.norm_scale)) \
        if warm is not None else None
    data = gather_expert_data_device(grid, dgrid, sub, scale, norm=norm) if dgrid is not None \
        else gather_expert_data(grid, sub, scale, norm=norm)
    expert = EncodedSubdomain(id=sub.id, cell=sub.cell, cluster_id=sub.cluster_id, norm_origin=data.norm_origin,
                              norm_scale=data.norm_scale, value_scale=scale)
    inputs = {"l1": (data.l1_inputs, data.l1_labels), "tile": (data.tile_inputs, data.tile_targets),
              "l0": (data.l0_inputs, data.l0_labels), "voxel": (data.vox_inputs, data.vox_targets)}
    jobs = []
    for tag, attr in _EXPERT_NETS:
        x, y = inputs[tag]
        spec = net_spec(tag, cfg)
        if spec is None or x is None:
            if x is not None and spec is None and tag == "tile":
                logger.warning("expert %d: active tiles present but config has no tile network", sub.id)
            continue
        warm_net = dict(warm.nets()).get(tag) if warm is not None else None
        stop = None if stop_losses is None else stop_losses.get(tag)
        try:
            tr, ff = make_trainer(x, y, spec, cfg, sub.id, lr0, warm=warm_net, stop_loss=stop, device=device,
                                  group=group)
        except Exception as exc:
            raise EncodeError(f"{tag} training failed: {exc}", sub.id) from exc
        jobs.append((attr, tr, ff))
    return expert, jobs


def _train_experts(grid: DenseLeafGrid, subs, cfg, lr0: float, warm_of, stops_of, device=None, group=None,
                   dgrid: Optional[DeviceGrid] = None):
    """Train every net of every given expert: an expert's nets run at once on
    their own streams, each with its full grid (``run_concurrent``; splitting
    the SMs between them instead was measured slower, because the epoch
    kernels are latency-bound per tile and a smaller share lengthens each
    CTA's tile chain)."""
    experts = []
    if dgrid is None and subs:
        dgrid = DeviceGrid(grid, device)  # training sets gathered on the device
    for sub in subs:
        expert, jobs = _prepare_expert(grid, sub, cfg, lr0, warm=warm_of(sub), stop_losses=stops_of(sub),
                                       device=device, group=group, dgrid=dgrid)
        try:
            for (attr, tr, ff), (loss, epochs) in zip(jobs, run_concurrent([tr for _, tr, _ in jobs])):
                setattr(expert, attr, NetRecord(params=tr.weights(), ff=ff, final_loss=float(loss), epochs=epochs))
        finally:
            for _, tr, _ in jobs:
                tr.close()
        if expert.voxel_regressor is None:
            logger.warning("expert %d: no active voxels, value regressor skipped", expert.id)
        experts.append(expert)
    return experts


def encode(grid, cfg, weight_precision: int = 32, workers: int = 1, _warm=None, _lr0=None, _stop_losses=None,
           device=None, group=None) -> NeuralGridContainer:
    """Encode a grid into its hierarchical neural container (encoder.py:573-611).

    ``group``: a ``torch.distributed`` group of G > 1 ranks, one per GPU, all
    calling with the same grid (SURVEY.md §8(e) "Training").  With at least G
    experts the experts are spread round-robin over the ranks (independent,
    no collective while training; the reference's expert thread pool,
    encoder.py:596-600) and each rank extracts its experts' patches; the
    trained experts are then exchanged so every rank returns the complete
    container.  With fewer experts than ranks every network is trained data
    parallel (each rank a 1/G slice of every epoch's batch, one packed
    gradient + loss all-reduce per epoch)."""
    del workers  # experts train one after another on the device; each net uses the whole GPU
    _validate(cfg)
    g = as_grid(grid)
    layout = decompose(g, cfg.subdomain_size)
    if not layout.subdomains:
        raise EncodeError("grid has no active values")
    lr0 = cfg.lr if _lr0 is None else _lr0
    world, rank = 1, 0
    if group is not None:
        import torch.distributed as dist
        world, rank = dist.get_world_size(group), dist.get_rank(group)
    expert_parallel = world > 1 and len(layout.subdomains) >= world
    dp_group = group if world > 1 and not expert_parallel else None
    mine_subs = [sub for i, sub in enumerate(layout.subdomains) if not expert_parallel or i % world == rank]

    def warm_of(sub):
        return _warm.get(sub.cell) if _warm else None

    def stops_of(sub):
        if _stop_losses is None:
            return None
        return {tag: _stop_losses[(sub.cell, tag)] for tag in NET_TAGS if (sub.cell, tag) in _stop_losses}

    dgrid = DeviceGrid(g, device)  # the grid on the device once: training sets and patch extraction
    experts = _train_experts(g, mine_subs, cfg, lr0, warm_of, stops_of, device=device, group=dp_group, dgrid=dgrid)
    if expert_parallel:
        # every rank needs all experts: patch extraction blends across
        # subdomain boundaries and the container holds every expert
        import torch.distributed as dist
        got: list = [None] * world
        dist.all_gather_object(got, experts, group=group)
        experts = sorted((e for part in got for e in part), key=lambda e: e.id)
        mine = [s.id for i, s in enumerate(layout.subdomains) if i % world == rank]
        extract_patches(g, layout, experts, cfg, device, only=set(mine), dgrid=dgrid)
        pats: list = [None] * world
        dist.all_gather_object(pats, {e.id: e.patches for e in experts if e.id in mine}, group=group)
        by_id = {e.id: e for e in experts}
        for part in pats:
            for sid, p in part.items():
                by_id[sid].patches = p
    else:
        extract_patches(g, layout, experts, cfg, device, dgrid=dgrid)
    del dgrid
    meta = GridMeta(g.grid_class, g.background, g.voxel_size, g.half_width, value_scale_of(g))
    return NeuralGridContainer(grid_meta=meta, upper_tree=build_upper_tree(g), layout=layout, experts=experts,
                               config=replace(cfg) if hasattr(cfg, "__dataclass_fields__") else cfg,
                               weight_precision=weight_precision)


@dataclass
class FrameReport:
    """encoder.py:617-624."""

    frame: int
    epochs: int
    final_loss: float
    detail: Dict[str, float] = field(default_factory=dict)


def _frame_epochs(c) -> int:
    return sum(net.epochs for e in c.experts for _, net in e.nets() if net is not None)


def _frame_loss(c) -> float:
    losses = [e.voxel_regressor.final_loss for e in c.experts if e.voxel_regressor is not None]
    return float(np.mean(losses)) if losses else 0.0


def encode_sequence(grids: Sequence, cfg, weight_precision: int = 32, workers: int = 1, device=None, group=None):
    """Warm-start encoding of an animated sequence (encoder.py:638-714)."""
    if len(grids) < 2:
        raise EncodeError("a sequence needs at least 2 frames")
    gs = [as_grid(g) for g in grids]
    for i, g in enumerate(gs[1:], start=1):
        if g.voxel_size != gs[0].voxel_size:
            raise EncodeError(f"frame {i}: voxel size {g.voxel_size} != {gs[0].voxel_size}")
        if g.grid_class != gs[0].grid_class:
            raise EncodeError(f"frame {i}: grid class mismatch")
    refine_lr = cfg.refine_lr if cfg.refine_lr is not None else cfg.lr
    containers, reports = [], []
    targets: Dict[Tuple[Tuple[int, int, int], str], float] = {}

    def frame_cfg(pass_id: int):
        return replace(cfg, seed=stable_seed(cfg.seed, 9000 + pass_id))

    def cold_refine(g, pass_id, warm_from=None, only_cells=None):
        cold = encode(g, frame_cfg(pass_id), weight_precision, workers, _warm=warm_from, device=device, group=group)
        cold_epochs = _frame_epochs(cold)
        warm = {e.cell: e for e in cold.experts if only_cells is None or e.cell in only_cells}
        refined = encode(g, frame_cfg(pass_id + 1), weight_precision, workers, _warm=warm, _lr0=refine_lr,
                         device=device, group=group)
        return cold, refined, cold_epochs

    _, frame0, cold_epochs0 = cold_refine(gs[0], 0)
    for e in frame0.experts:
        for tag, net in e.nets():
            if net is not None:
                targets[(e.cell, tag)] = net.final_loss
    containers.append(frame0)
    reports.append(FrameReport(0, cold_epochs0 + _frame_epochs(frame0), _frame_loss(frame0),
                               {"cold_epochs": float(cold_epochs0), "refine_epochs": float(_frame_epochs(frame0))}))
    prev = frame0
    for t in range(1, len(gs)):
        prev_by_cell = {e.cell: e for e in prev.experts}
        layout_t = decompose(gs[t], cfg.subdomain_size)
        new_cells = [s.cell for s in layout_t.subdomains if s.cell not in prev_by_cell]
        warm = dict(prev_by_cell)
        if new_cells:
            _, refined_t, _ = cold_refine(gs[t], 10 * t)
            for e in refined_t.experts:
                if e.cell in new_cells:
                    warm[e.cell] = e
                    for tag, net in e.nets():
                        if net is not None:
                            targets[(e.cell, tag)] = net.final_loss
        ct = encode(gs[t], frame_cfg(10 * t + 2), weight_precision, workers, _warm=warm, _lr0=refine_lr,
                    _stop_losses=targets, device=device, group=group)
        containers.append(ct)
        reports.append(FrameReport(t, _frame_epochs(ct), _frame_loss(ct), {}))
        prev = ct
    return containers, reports
