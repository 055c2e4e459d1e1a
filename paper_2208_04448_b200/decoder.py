"""Whole-volume decode and the random-access hybrid grid on the GPU.

Drop-in for ``decoder.decode_full`` / ``make_hybrid`` / ``HybridGrid.query``
(decoder.py:101-270).  The host sequences the C-ABI primitives in the same
order as the reference's ``_reconstruct`` / ``_fill_leaves``; all per-point
work (classification, regression, blending, patches, fills) runs in the CUDA
kernels of ``csrc/``.  Node indexing follows the reference: level-1 nodes in
sorted-origin order (decoder.py:71), leaves in node order x ascending slot
(decoder.py:146-151).
"""

from __future__ import annotations

import ctypes as C
import itertools
import sys
from dataclasses import dataclass
from typing import Dict, Optional, Tuple

import numpy as np
import torch

from . import _lib
from ._lib import EvalOut, check, lib
from .errors import SvcodecError
from .model import (L1_SIZE, L2_SIZE, LEAF_SIZE, DenseLeafGrid, L1TileMap, LeafBitsMap, PatchRecords)
from .netset import TAG_CODES, DeviceNetSet
from .tree import DeviceTree

EVAL_CHUNK = 1 << 24  # points per evaluator call on the multi-expert path
MAX_CALL = 1 << 30    # points per evaluator call on the single-expert path (int32 tile counts)
PIPE_LEAVES = 1024    # decode_full's pipelined voxel stage: leaf ranges of at least this many leaves


def _dev(device=None) -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2208_04448_b200 needs a CUDA device (no CPU fallback)")
    return torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())


def _stream(dev):
    return torch.cuda.current_stream(dev).cuda_stream


def _ptr(t: Optional[torch.Tensor], byte_offset: int = 0):
    return None if t is None else t.data_ptr() + byte_offset


class _PinnedPool:
    """Reusable pinned host blocks for decode and query outputs.  A block is
    handed out as numpy views of one pooled uint8 array; it is free again once
    every view a caller holds is gone (reference count of the pooled array) and
    its last host->device copy has completed.  A full pool replaces its least
    recently used free block, so blocks that callers keep (results of the
    previous call) never force an uncached cudaHostAlloc per call."""

    CAP = 12

    def __init__(self):
        self.blocks = []  # [pinned uint8 tensor, its numpy view, fence event, last use]
        self.clock = 0

    @staticmethod
    def _idle(blk) -> bool:
        # held by blk + getrefcount's argument only; its last host->device copy done
        return sys.getrefcount(blk[1]) <= 2 and (blk[2] is None or blk[2].query())

    def get(self, nbytes: int):
        self.clock += 1
        free = [blk for blk in self.blocks if blk[1].size >= nbytes and self._idle(blk)]
        if free:
            blk = min(free, key=lambda b: b[1].size)  # best fit
            blk[2] = None
            blk[3] = self.clock
            return blk[0], blk[1]
        if len(self.blocks) >= self.CAP:
            idle = [blk for blk in self.blocks if self._idle(blk)]
            if idle:
                self.blocks.remove(min(idle, key=lambda b: b[3]))
        t = torch.empty(max(nbytes, 1 << 20), dtype=torch.uint8, pin_memory=True)
        blk = [t, t.numpy(), None, self.clock]
        if len(self.blocks) < self.CAP:
            self.blocks.append(blk)
        return blk[0], blk[1]

    def fence(self, arr, event) -> None:
        """The block behind ``arr`` is the source of a copy completing at ``event``."""
        for blk in self.blocks:
            if blk[1] is arr:
                blk[2] = event


_PINNED = _PinnedPool()
_SIDE_STREAMS: Dict[int, "torch.cuda.Stream"] = {}


def _to_host(ts):
    """Device tensors -> numpy arrays over one pinned host block: asynchronous
    copies on the current stream, one synchronize."""
    offs, n = [], 0
    for t in ts:
        offs.append(n)
        n += (t.numel() * t.element_size() + 255) & ~255
    blk = _PINNED.get(n)
    pin, arr = blk
    outs = []
    for t, o in zip(ts, offs):
        nb = t.numel() * t.element_size()
        pin[o:o + nb].view(t.dtype).view(t.shape).copy_(t, non_blocking=True)
        outs.append(arr[o:o + nb].view(_NP_DTYPE[t.dtype]).reshape(tuple(t.shape)))
    if ts:
        torch.cuda.current_stream(ts[0].device).synchronize()
    return outs


_COPY_POOL = None


def _to_device(a: np.ndarray, dev) -> torch.Tensor:
    """Host array -> device tensor through a pooled pinned block, in 32 MiB
    pieces: each piece's pageable -> pinned copy is split over host threads
    (numpy releases the GIL while copying) and its asynchronous host->device
    copy on the current stream runs while the next piece is staged.  The
    block is fenced until the last copy completes."""
    global _COPY_POOL
    a = np.ascontiguousarray(a)
    n = a.nbytes
    if n < (8 << 20):  # small: the driver's staged copy is as fast
        return torch.from_numpy(a).to(dev)
    pin, arr = _PINNED.get(n)
    src = a.reshape(-1).view(np.uint8)
    out = torch.empty(a.shape, dtype=_TORCH_DTYPE[a.dtype.type], device=dev)
    obytes = out.view(-1).view(torch.uint8)
    if _COPY_POOL is None:
        from concurrent.futures import ThreadPoolExecutor
        _COPY_POOL = ThreadPoolExecutor(8, thread_name_prefix="nvdb-h2d")
    piece = 32 << 20
    for p0 in range(0, n, piece):
        p1 = min(n, p0 + piece)
        k = int(min(8, max(1, (p1 - p0) >> 22)))
        cuts = [p0 + (((p1 - p0) * i // k) & ~4095) for i in range(k)] + [p1]
        list(_COPY_POOL.map(lambda i: np.copyto(arr[cuts[i]:cuts[i + 1]], src[cuts[i]:cuts[i + 1]]), range(k)))
        obytes[p0:p1].copy_(pin[p0:p1], non_blocking=True)
    ev = torch.cuda.Event()
    ev.record(torch.cuda.current_stream(dev))
    _PINNED.fence(arr, ev)
    return out


_TORCH_DTYPE = {np.uint8: torch.uint8, np.int32: torch.int32, np.int64: torch.int64, np.float32: torch.float32}
_NP_DTYPE = {torch.uint8: np.uint8, torch.int32: np.int32, torch.int64: np.int64, torch.float32: np.float32,
             torch.float64: np.float64, torch.bool: np.bool_}


def _slot1(c) -> int:
    """idx1 of a coordinate (grid.py:74-94)."""
    return (((c[0] & 127) >> 3) << 8) | (((c[1] & 127) >> 3) << 4) | ((c[2] & 127) >> 3)


def _slot0(c) -> int:
    return ((c[0] & 7) << 6) | ((c[1] & 7) << 3) | (c[2] & 7)


def _slot1_arr(k: np.ndarray) -> np.ndarray:
    return (((k[:, 0] & 127) >> 3) << 8) | (((k[:, 1] & 127) >> 3) << 4) | ((k[:, 2] & 127) >> 3)


def _slot0_arr(k: np.ndarray) -> np.ndarray:
    return ((k[:, 0] & 7) << 6) | ((k[:, 1] & 7) << 3) | (k[:, 2] & 7)


def _patch_arrays(lists, nfields: int):
    """Concatenate the experts' patch lists [(coord, f1[, f2])] into arrays;
    a key repeated by a later expert overrides the earlier one (decoder.py:84-92)."""
    keys, fields = [np.zeros((0, 3), np.int64)], [[np.zeros(0)] for _ in range(nfields)]
    for lst in lists:
        if not len(lst):
            continue
        if isinstance(lst, PatchRecords):  # columns already (model.PatchRecords)
            k, *cs = lst.arrays()
            keys.append(k)
            for f in range(nfields):
                fields[f].append(cs[f].astype(np.float64))
            continue
        n = len(lst)
        cols = list(zip(*lst))
        keys.append(np.fromiter(itertools.chain.from_iterable(cols[0]), dtype=np.int64, count=3 * n).reshape(-1, 3))
        for f in range(nfields):
            fields[f].append(np.fromiter(cols[1 + f], dtype=np.float64, count=n))
    k = np.concatenate(keys)
    fs = [np.concatenate(fl) for fl in fields]
    if sum(1 for lst in lists if len(lst)) > 1 and k.shape[0]:
        # keep the last occurrence of each key, in first-occurrence order of the kept rows
        _, first_rev = np.unique(k[::-1], axis=0, return_index=True)
        last = np.sort(k.shape[0] - 1 - first_rev)
        k = k[last]
        fs = [f[last] for f in fs]
    if nfields == 1:
        return k, fs[0].astype(np.int64)
    return k, fs[0].astype(bool), fs[1]


class NetEvaluator:
    """Experts' nets on the GPU plus the generic gate-blended evaluator."""

    def __init__(self, experts, subdomain_size: int, halo: int, background: float = 0.0, device=None):
        self.dev = _dev(device)
        self.background = float(np.float32(background))
        experts = sorted(experts, key=lambda e: e.id)
        self.ns = DeviceNetSet(experts, subdomain_size, halo, device=self.dev)
        self.single = len(experts) == 1
        self.has_tag = {t: any(dict(e.nets()).get(t) is not None for e in experts) for t in TAG_CODES}

    def close(self):
        self.ns.close()

    def evaluate(self, tag: str, src_kind: int, src: torch.Tensor, n: int, out_mode: int, *,
                 gather: Optional[torch.Tensor] = None, u8=None, f32=None, probs=None, raw=None,
                 value_scale: float = 1.0, clip: bool = False, count: Optional[torch.Tensor] = None) -> None:
        return DeviceModel.evaluate(self, tag, src_kind, src, n, out_mode, gather=gather, u8=u8, f32=f32,
                                    probs=probs, raw=raw, value_scale=value_scale, clip=clip, count=count)

    def select(self, v: torch.Tensor, value: int, sync: bool = True):
        return DeviceModel.select(self, v, value, sync)


class DeviceModel:
    """A container prepared for decoding: nets, node origins and patch tables on the GPU."""

    def __init__(self, c, device=None):
        self.c = c
        self.dev = _dev(device)
        meta = c.grid_meta
        self.meta = meta
        self.background = float(np.float32(meta.background))
        self.value_scale = float(meta.value_scale)
        experts = sorted(c.experts, key=lambda e: e.id)
        self.ns = DeviceNetSet(experts, c.layout.size, c.layout.halo, device=self.dev)
        self.single = len(experts) == 1
        self.has_tag = {t: any(dict(e.nets()).get(t) is not None for e in experts) for t in TAG_CODES}
        ut = c.upper_tree
        # level-1 origins validated against level-2 child bits (decoder.py:66-77)
        l2 = {tuple(int(v) for v in n.origin): n for n in ut.l2_nodes}
        expected = sum(int(np.count_nonzero(n.child_mask.bits)) for n in ut.l2_nodes)
        if expected != len(ut.l1_origins):
            raise SvcodecError(f"corrupt container: {len(ut.l1_origins)} level-1 origins vs "
                               f"{expected} level-2 child bits")
        origins = sorted(tuple(int(v) for v in o) for o in ut.l1_origins)
        for o in origins:
            root = tuple(v & ~4095 for v in o)
            idx2 = (((o[0] & 4095) >> 7) << 10) | (((o[1] & 4095) >> 7) << 5) | ((o[2] & 4095) >> 7)
            n2 = l2.get(root)
            if n2 is None or not n2.child_mask.bits[idx2]:
                raise SvcodecError(f"corrupt container: level-1 origin {o} has no level-2 child bit")
        self.origins = np.asarray(origins, dtype=np.int64).reshape(-1, 3)
        self.n1 = len(origins)
        host = {"d_origins": self.origins.astype(np.int32)}  # device tables, uploaded together below
        # dense node table over the origins' bounding box: patch / fill / tile
        # coordinates become node * 4096 + idx1 on the device (nvdb_node_slots)
        self._lut_lo = self._lut_span = None
        if self.n1:
            o = self.origins >> 7
            lo, span = o.min(axis=0), o.max(axis=0) - o.min(axis=0) + 1
            if float(span[0]) * float(span[1]) * float(span[2]) <= float(1 << 24) and (np.abs(self.origins) < (1 << 30)).all():
                code = ((o[:, 0] - lo[0]) * span[1] + (o[:, 1] - lo[1])) * span[2] + (o[:, 2] - lo[2])
                lut = np.full(int(span.prod()), -1, np.int32)
                lut[code[::-1]] = np.arange(self.n1, dtype=np.int32)[::-1]
                host["lut"] = lut
                self._lut_lo = (C.c_int32 * 3)(*[int(v) for v in lo])
                self._lut_span = (C.c_int32 * 3)(*[int(v) for v in span])
        # patch maps (decoder.py:84-92): later experts override earlier keys
        l1k, l1c = _patch_arrays([e.patches.l1 for e in c.experts], 1)
        host["p1_key"] = l1k.astype(np.int32).reshape(-1, 3)
        host["p1_cls"] = np.asarray(l1c).astype(np.uint8)
        # tile records per level-1 node
        t_slot, t_val = self._tile_records(ut.l1_tiles)
        host["t_slot"], host["t_val"] = t_slot, t_val
        host["err"] = np.zeros(2, np.int32)  # [0] level-1 patch outside every node
        self._tables = []
        self._upload(host)
        self.p1_slot = torch.empty(max(l1k.shape[0], 1), dtype=torch.int64, device=self.dev)[:l1k.shape[0]]
        self._slots(self.p1_key, self.p1_slot, None, self.err[:1], "level-1 patch")
        self._l0_ready = False  # level-0 tables: built by _ensure_l0 (decode overlaps them with the L0 stage)

    def _slots(self, keys: torch.Tensor, slot: torch.Tensor, vox, err, what: str) -> None:
        """node * 4096 + idx1 (and idx0) of int32 coordinate rows, on the device."""
        n = keys.shape[0]
        if n == 0:
            return
        if self._lut_lo is not None:
            check(lib().nvdb_node_slots(_ptr(self.lut), self._lut_lo, self._lut_span, _ptr(keys), n, _ptr(slot),
                                        _ptr(vox), _ptr(err), _stream(self.dev)), "nvdb_node_slots")
            return
        # very sparse node sets (bounding box > 2^24 cells): host lookup
        k = keys.cpu().numpy().astype(np.int64)
        ni = self._node_index(k & ~np.int64(127))
        if err is not None and (ni < 0).any():
            err.fill_(1)
        slot.copy_(torch.from_numpy(np.where(ni < 0, -1, ni * L1_SIZE + _slot1_arr(k)).astype(np.int64)))
        if vox is not None:
            vox.copy_(torch.from_numpy(_slot0_arr(k).astype(np.int32)))

    def _tile_records(self, tiles_map):
        """(slot, value) of the inactive-tile records (decoder.py:126-134); an
        unknown node raises SvcodecError (decoder.py:128-130)."""
        if isinstance(tiles_map, L1TileMap):  # columns already (model.L1TileMap)
            torg, counts, slots, vals = tiles_map.arrays()
        else:
            torg = np.asarray(list(tiles_map.keys()), dtype=np.int64).reshape(-1, 3)
            ds = list(tiles_map.values())
            counts = np.fromiter((len(d) for d in ds), dtype=np.int64, count=len(ds))
            slots = np.fromiter(itertools.chain.from_iterable(d.keys() for d in ds), dtype=np.int64,
                                count=int(counts.sum()))
            vals = np.fromiter(itertools.chain.from_iterable(d.values() for d in ds), dtype=np.float32,
                               count=int(counts.sum()))
        if torg.shape[0] == 0:
            return np.zeros(0, np.int64), np.zeros(0, np.float32)
        tni = self._node_index(torg)
        if (tni < 0).any():
            bad = tuple(int(v) for v in torg[int(np.flatnonzero(tni < 0)[0])])
            raise SvcodecError(f"corrupt container: tile record for unknown level-1 node {bad}")
        return (np.repeat(tni, counts) * L1_SIZE + slots).astype(np.int64), vals.astype(np.float32)

    def _ensure_l0(self, after: Optional[torch.cuda.Event] = None) -> None:
        """Level-0 patch and negative-fill tables (one upload; slots on the device).

        ``after``: an event on the current stream recorded before the level-0
        stage was enqueued; the upload and its slot kernels then run on the
        side stream beside that stage, and the current stream waits for them."""
        if self._l0_ready:
            return
        if after is not None:
            main = torch.cuda.current_stream(self.dev)
            side = self._side_stream()
            side.wait_event(after)
            with torch.cuda.stream(side):
                self._ensure_l0()
            for k in ("p0_key", "p0_act", "p0_val", "neg_key", "neg_u8", "p0_slot", "p0_vox", "neg_slot",
                      "neg_bits"):
                getattr(self, k).record_stream(main)
            ev = torch.cuda.Event()
            ev.record(side)
            main.wait_event(ev)
            return
        c, ut = self.c, self.c.upper_tree
        host = {}
        l0k, l0a, l0v = _patch_arrays([e.patches.l0 for e in c.experts], 2)
        host["p0_key"] = l0k.astype(np.int32).reshape(-1, 3)
        host["p0_act"] = np.asarray(l0a).astype(np.uint8)
        host["p0_val"] = l0v.astype(np.float32)
        self._l0_keys = l0k
        nf = ut.leaf_negative_fill
        if len(nf):
            if isinstance(nf, LeafBitsMap):  # columns already (model.LeafBitsMap)
                norg, bits = nf.arrays()
            else:
                norg = np.fromiter(itertools.chain.from_iterable(nf.keys()), dtype=np.int64,
                                   count=3 * len(nf)).reshape(-1, 3)
                bits = np.concatenate(list(nf.values()), axis=None)  # each entry flattened (C order)
                if bits.size != LEAF_SIZE * len(nf):
                    raise SvcodecError("corrupt container: negative-fill entry of the wrong size")
                bits = bits.astype(bool, copy=False).reshape(-1, LEAF_SIZE)
            host["neg_key"] = norg.astype(np.int32).reshape(-1, 3)
            host["neg_u8"] = np.ascontiguousarray(bits).view(np.uint8).reshape(-1, LEAF_SIZE)
        else:
            host["neg_key"] = np.zeros((0, 3), np.int32)
            host["neg_u8"] = np.zeros((0, LEAF_SIZE), np.uint8)
        self._upload(host)
        n0, nn = l0k.shape[0], self.neg_key.shape[0]
        self.p0_slot = torch.empty(max(n0, 1), dtype=torch.int64, device=self.dev)[:n0]
        self.p0_vox = torch.empty(max(n0, 1), dtype=torch.int32, device=self.dev)[:n0]
        self._slots(self.p0_key, self.p0_slot, self.p0_vox, None, "level-0 patch")  # -1: flagged by l0_apply
        self.neg_slot = torch.empty(max(nn, 1), dtype=torch.int64, device=self.dev)[:nn]
        self._slots(self.neg_key, self.neg_slot, None, None, "negative fill")  # -1: skipped (not a leaf)
        self.neg_bits = torch.empty((max(nn, 1), 8), dtype=torch.int64, device=self.dev)[:nn]
        if nn:
            check(lib().nvdb_pack_eq(_ptr(self.neg_u8), nn * 8, 1, _ptr(self.neg_bits), _stream(self.dev)),
                  "nvdb_pack_eq")
        self._l0_ready = True

    @property
    def l0_keys(self) -> np.ndarray:
        """(n, 3) level-0 patch coordinates after the later-expert override."""
        self._ensure_l0()
        return self._l0_keys

    def _upload(self, host: Dict[str, np.ndarray]) -> None:
        """All device tables in one host buffer and one host->device copy;
        each attribute is a typed view of the device buffer."""
        offs, n = {}, 0
        for k, a in host.items():
            offs[k] = n
            n += (a.nbytes + 255) & ~255
        # pinned staging from the decode pool (handed out again once the copy
        # has completed): an asynchronous copy, no host wait
        pin, buf = _PINNED.get(max(n, 256))
        for k, a in host.items():
            buf[offs[k]:offs[k] + a.nbytes] = np.ascontiguousarray(a).reshape(-1).view(np.uint8)
        dbuf = torch.empty(max(n, 256), dtype=torch.uint8, device=self.dev)
        dbuf.copy_(pin[:max(n, 256)], non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream(self.dev))
        _PINNED.fence(buf, ev)
        self._tables.append(dbuf)
        for k, a in host.items():
            t = dbuf[offs[k]:offs[k] + a.nbytes].view(_TORCH_DTYPE[a.dtype.type]).view(a.shape)
            setattr(self, k, t)

    def _node_index(self, keys: np.ndarray) -> np.ndarray:
        """Level-1 node index (sorted-origin order) of each node-origin row, -1 if none."""
        keys = np.asarray(keys, dtype=np.int64).reshape(-1, 3)
        out = np.full(keys.shape[0], -1, np.int64)
        if keys.shape[0] == 0 or self.n1 == 0:
            return out
        if getattr(self, "_nidx", None) is None:
            o = self.origins >> 7
            lo = o.min(axis=0)
            span = o.max(axis=0) - lo + 1
            dense = float(span[0]) * float(span[1]) * float(span[2]) < 2.0 ** 62
            if dense:
                oc = ((o[:, 0] - lo[0]) * span[1] + (o[:, 1] - lo[1])) * span[2] + (o[:, 2] - lo[2])
                order = np.argsort(oc, kind="stable")
                ncode = int(span[0]) * int(span[1]) * int(span[2])
                lut = None
                if ncode <= (1 << 24):  # small bounding box: direct table instead of a binary search
                    lut = np.full(ncode, -1, np.int64)
                    lut[oc[::-1]] = np.arange(self.n1)[::-1]  # first of any repeated origin wins
                self._nidx = (lo, span, oc[order], order, lut)
            else:
                self._nidx = ()
        if self._nidx:
            # dense code over the origins' bounding box; rows outside it have no node
            lo, span, ocs, order, lut = self._nidx
            # column-wise (reductions over a 3-wide axis are slow in numpy)
            kx, ky, kz = ((keys[:, a] >> 7) - lo[a] for a in range(3))
            inside = ((kx.astype(np.uint64) < np.uint64(span[0])) & (ky.astype(np.uint64) < np.uint64(span[1]))
                      & (kz.astype(np.uint64) < np.uint64(span[2]))
                      & (((keys[:, 0] | keys[:, 1] | keys[:, 2]) & 127) == 0))
            kc = ((kx[inside] * span[1] + ky[inside]) * span[2] + kz[inside])
            if lut is not None:
                out[inside] = lut[kc]
                return out
            pos = np.minimum(np.searchsorted(ocs, kc), self.n1 - 1)
            hit = ocs[pos] == kc
            out[np.flatnonzero(inside)[hit]] = order[pos[hit]]
            return out
        allk = np.concatenate([self.origins, keys])
        _, inv = np.unique(allk, axis=0, return_inverse=True)
        inv = inv.reshape(-1)
        lut = np.full(inv.max() + 1, -1, np.int64)
        lut[inv[:self.n1]] = np.arange(self.n1)
        return lut[inv[self.n1:]]

    def _i64(self, xs):
        return torch.from_numpy(np.ascontiguousarray(xs, dtype=np.int64)).to(self.dev)

    def _u8(self, xs):
        return torch.from_numpy(np.ascontiguousarray(xs, dtype=np.uint8)).to(self.dev)

    def close(self):
        self.ns.close()

    # -- primitives --------------------------------------------------------------

    def evaluate(self, tag: str, src_kind: int, src: torch.Tensor, n: int, out_mode: int, *,
                 gather: Optional[torch.Tensor] = None, u8=None, f32=None, probs=None, raw=None,
                 value_scale: float = 1.0, clip: bool = False, count: Optional[torch.Tensor] = None) -> None:
        """nvdb_eval over n points, chunked on the multi-expert path.

        ``count``: a device int64 scalar; only its first ``count`` of the n
        (capacity) points are evaluated and n never has to visit the host
        (nvdb_eval_counted; single-expert nets only -- the blended path sizes
        its candidate passes on the host)."""
        if n == 0:
            return
        fast = self.single and self.has_tag[tag]
        if count is not None:
            if not fast or n > MAX_CALL:
                n = int(count.item())
                if n == 0:
                    return
            else:
                out = EvalOut(out_mode=out_mode, raw=_ptr(raw), probs=_ptr(probs), u8=_ptr(u8), f32=_ptr(f32),
                              value_scale=float(value_scale), background=self.background, clip=int(bool(clip)))
                timer = getattr(self, "timer", None)
                if timer is not None:
                    ev0 = torch.cuda.Event(enable_timing=True)
                    ev1 = torch.cuda.Event(enable_timing=True)
                    ev0.record()
                check(lib().nvdb_eval_counted(self.ns.handle, TAG_CODES[tag], src_kind, _ptr(src), _ptr(gather), n,
                                              _ptr(count), C.byref(out), None, 0, _stream(self.dev)),
                      "nvdb_eval_counted")
                if timer is not None:
                    ev1.record()
                    timer.append((tag, count, ev0, ev1))
                return
        chunk = min(n, MAX_CALL) if fast else EVAL_CHUNK
        if src_kind == _lib.SRC_LEAF_VOX and gather is None:
            chunk = max(512, chunk // 512 * 512)
        if src_kind == _lib.SRC_L1_SLOT and gather is None:
            chunk = max(4096, chunk // 4096 * 4096)
        k = 3 if tag == "l1" else 1
        ws = None
        if not fast:
            wsb = lib().nvdb_eval_workspace_bytes(self.ns.handle, min(chunk, n))
            ws = torch.empty(max(int(wsb), 1), dtype=torch.uint8, device=self.dev)
        st = _stream(self.dev)
        timer = getattr(self, "timer", None)
        for s in range(0, n, chunk):
            m = min(chunk, n - s)
            if timer is not None:
                ev0 = torch.cuda.Event(enable_timing=True)
                ev1 = torch.cuda.Event(enable_timing=True)
                ev0.record()
            if gather is not None:
                g, sp = _ptr(gather, 8 * s), _ptr(src)
            else:
                g = None
                per = {_lib.SRC_LEAF_VOX: (512, 12), _lib.SRC_L1_SLOT: (4096, 12),
                       _lib.SRC_COORD_I32: (1, 12), _lib.SRC_CENTER_F64: (1, 24),
                       _lib.SRC_NORM_F32: (1, 12)}[src_kind]
                sp = _ptr(src, (s // per[0]) * per[1])
            out = EvalOut(out_mode=out_mode,
                          raw=_ptr(raw, 4 * k * s), probs=_ptr(probs, 8 * k * s),
                          u8=_ptr(u8, s), f32=_ptr(f32, 4 * s), value_scale=float(value_scale),
                          background=self.background, clip=int(bool(clip)))
            check(lib().nvdb_eval(self.ns.handle, TAG_CODES[tag], src_kind, sp, g, m, C.byref(out),
                                  _ptr(ws), 0 if ws is None else ws.numel(), st), "nvdb_eval")
            if timer is not None:
                ev1.record()
                timer.append((tag, m, ev0, ev1))

    def select(self, v: torch.Tensor, value: int, sync: bool = True):
        """ids of v == value, ascending.  sync: one device->host count read,
        returns the ids; otherwise returns (ids at capacity v.numel(), device
        int64 count) without a host round trip."""
        n = v.numel()
        ids = torch.empty(max(n, 1), dtype=torch.int64, device=self.dev)
        cnt = torch.zeros(1, dtype=torch.int64, device=self.dev)
        wsb = lib().nvdb_select_workspace_bytes(n)
        ws = torch.empty(int(wsb), dtype=torch.uint8, device=self.dev)
        check(lib().nvdb_select_u8(_ptr(v), n, value, _ptr(ids), _ptr(cnt), _ptr(ws), ws.numel(),
                                   _stream(self.dev)), "nvdb_select_u8")
        if not sync:
            return ids, cnt
        return ids[:int(cnt.item())]

    # -- decode --------------------------------------------------------------------

    def decode(self, materialize_values: bool = True, shard: Optional[Tuple[int, int]] = None,
               prefetch_host: bool = False) -> "DeviceDecode":
        """decoder._reconstruct (decoder.py:101-211) on the device.

        ``shard=(rank, world)``: level-1 classification runs on every rank
        (n1*4096 slots, cheap), then the leaf list is split into ``world``
        contiguous ranges (:func:`shard_range`) and this rank classifies,
        regresses and finalizes only its own leaves -- no collective.

        ``prefetch_host=True`` (``decode_full``): the arrays that are final
        once the level-0 patches are applied (level-1 classes and tiles, leaf
        origins, active flags) are copied to pinned host memory on a side
        stream while the voxel stage runs; ``to_grid`` then copies only the
        values.
        """
        dev, st = self.dev, _stream(self.dev)
        n1 = self.n1
        nslots = n1 * L1_SIZE
        cls = torch.empty(max(nslots, 1), dtype=torch.uint8, device=dev)
        tiles = torch.full((max(nslots, 1),), self.background, dtype=torch.float32, device=dev)
        self.evaluate("l1", _lib.SRC_L1_SLOT, self.d_origins, nslots, _lib.OUT_L1CLASS, u8=cls)
        check(lib().nvdb_l1_apply(_ptr(cls), _ptr(tiles), nslots, _ptr(self.p1_slot), _ptr(self.p1_cls),
                                  self.p1_slot.numel(), _ptr(self.t_slot), _ptr(self.t_val), self.t_slot.numel(),
                                  st), "nvdb_l1_apply")
        # active tiles through the tile regressor; without a tile net they stay
        # background (blended_values uncovered -> background, decoder.py:135-141)
        if self.has_tag["tile"]:
            tids, tcnt = self.select(cls[:nslots], 1, sync=False)
            tv = torch.empty(max(nslots, 1), dtype=torch.float32, device=dev)
            # tile values scale by float(np.float32(value_scale)), no clip (decoder.py:141)
            self.evaluate("tile", _lib.SRC_L1_SLOT, self.d_origins, nslots, _lib.OUT_VALUE, gather=tids, f32=tv,
                          value_scale=float(np.float32(self.value_scale)), count=tcnt)
            check(lib().nvdb_scatter_f32_counted(_ptr(tiles), _ptr(tids), _ptr(tv), nslots, _ptr(tcnt), st),
                  "nvdb_scatter_f32_counted")
        # the one host round trip of a decode: the leaf count sizes the leaf buffers
        child = self.select(cls[:nslots], 0)
        leaf_of_slot = torch.empty(max(nslots, 1), dtype=torch.int32, device=dev)
        if shard is not None:
            # global slot -> leaf map, then keep this rank's range; other ranks'
            # leaves are marked -2 (skipped, not an error) in the patch kernels
            lo, hi = shard_range(child.numel(), *shard)
            full = torch.empty((max(child.numel(), 1), 3), dtype=torch.int32, device=dev)
            check(lib().nvdb_leaf_list(_ptr(child), child.numel(), _ptr(self.d_origins), nslots, _ptr(full),
                                       _ptr(leaf_of_slot), st), "nvdb_leaf_list")
            loc = leaf_of_slot - lo
            leaf_of_slot = torch.where(leaf_of_slot < 0, leaf_of_slot,
                                       torch.where((loc >= 0) & (loc < hi - lo), loc, torch.full_like(loc, -2)))
            child = child[lo:hi]
            leaf_origins = full[lo:hi].contiguous() if hi > lo else full[:1]
            nl = hi - lo
        else:
            nl = child.numel()
            leaf_origins = torch.empty((max(nl, 1), 3), dtype=torch.int32, device=dev)
            check(lib().nvdb_leaf_list(_ptr(child), nl, _ptr(self.d_origins), nslots, _ptr(leaf_origins),
                                       _ptr(leaf_of_slot), st), "nvdb_leaf_list")
        nv = nl * LEAF_SIZE
        act = torch.zeros(max(nv, 1), dtype=torch.uint8, device=dev)
        pre_l0 = None
        if not self._l0_ready:
            pre_l0 = torch.cuda.Event()
            pre_l0.record(torch.cuda.current_stream(dev))
        self.evaluate("l0", _lib.SRC_LEAF_VOX, leaf_origins, nv, _lib.OUT_L0ACTIVE, u8=act)
        self._ensure_l0(after=pre_l0)  # host work and the table upload while the L0 stage runs
        err = torch.zeros(1, dtype=torch.int32, device=dev)
        check(lib().nvdb_l0_apply(_ptr(act), _ptr(self.p0_slot), _ptr(self.p0_vox), _ptr(self.p0_act),
                                  self.p0_slot.numel(), _ptr(leaf_of_slot), _ptr(err), st), "nvdb_l0_apply")
        pre = None
        if prefetch_host and shard is None and nl:
            pre = self._host_prefetch([cls[:nslots], tiles[:nslots], leaf_origins[:nl], act[:nv], err,
                                      self.err])
        act_ids = vals = None
        acnt = torch.zeros(1, dtype=torch.int64, device=dev)
        if (pre is not None and materialize_values and nl >= 4 * PIPE_LEAVES
                and self.single and self.has_tag["voxel"]):
            d = self._decode_pipelined(cls, tiles, child, leaf_origins, leaf_of_slot, act, nl, err, shard)
            d.host_pre = pre
            return d
        if materialize_values and nl:
            # active voxels -> voxel regressor -> finalize, the count staying on the device
            act_ids, acnt = self.select(act[:nv], 1, sync=False)
            vals = torch.empty(max(nv, 1), dtype=torch.float32, device=dev)
            self.evaluate("voxel", _lib.SRC_LEAF_VOX, leaf_origins, nv, _lib.OUT_VALUE, gather=act_ids,
                          f32=vals, value_scale=self.value_scale, clip=self.meta.grid_class == "sdf", count=acnt)
        values = torch.empty(max(nv, 1), dtype=torch.float32, device=dev)
        words = torch.empty(max(nl * 8, 1), dtype=torch.int64, device=dev)
        patched = torch.empty(max(nv, 1), dtype=torch.uint8, device=dev)
        check(lib().nvdb_leaf_finalize_counted(nl, _ptr(act), _ptr(act_ids), _ptr(vals),
                                               nv if act_ids is not None else 0, _ptr(acnt), _ptr(self.p0_slot),
                                               _ptr(self.p0_vox), _ptr(self.p0_act), _ptr(self.p0_val),
                                               self.p0_slot.numel(), _ptr(self.neg_slot), _ptr(self.neg_bits),
                                               self.neg_slot.numel(), _ptr(leaf_of_slot), self.background,
                                               -float(np.float32(self.value_scale)), _ptr(values), _ptr(words),
                                               _ptr(patched), st), "nvdb_leaf_finalize_counted")
        d = DeviceDecode(self, cls[:nslots], tiles[:nslots], child, leaf_origins[:nl], act[:nv],
                         values[:nv], words[:nl * 8], patched[:nv], acnt, shard, err)
        d.host_pre = pre
        if pre is not None:
            # the dense values follow on the copy stream as soon as finalize is
            # done; to_grid orders the leaves on the host while they travel
            d.host_vals = self._host_prefetch([values[:nv]])
        return d

    def _decode_pipelined(self, cls, tiles, child, leaf_origins, leaf_of_slot, act, nl, err, shard):
        """Voxel stage + value scatter in leaf ranges, each range's dense values
        copied to pinned host memory (copy stream) while the next range is
        regressed.  Finalize runs first without the regressor values (fills,
        patches, negative fill, masks); the per-range scatter skips patched
        voxels, so every value equals the one-pass decode's."""
        dev, st = self.dev, _stream(self.dev)
        nv = nl * LEAF_SIZE
        values = torch.empty(nv, dtype=torch.float32, device=dev)
        words = torch.empty(nl * 8, dtype=torch.int64, device=dev)
        patched = torch.empty(nv, dtype=torch.uint8, device=dev)
        zero = torch.zeros(1, dtype=torch.int64, device=dev)
        check(lib().nvdb_leaf_finalize_counted(nl, _ptr(act), None, None, 0, _ptr(zero), _ptr(self.p0_slot),
                                               _ptr(self.p0_vox), _ptr(self.p0_act), _ptr(self.p0_val),
                                               self.p0_slot.numel(), _ptr(self.neg_slot), _ptr(self.neg_bits),
                                               self.neg_slot.numel(), _ptr(leaf_of_slot), self.background,
                                               -float(np.float32(self.value_scale)), _ptr(values), _ptr(words),
                                               _ptr(patched), st), "nvdb_leaf_finalize_counted")
        cs = self._side_stream()
        pin, arr = _PINNED.get(nv * 4)
        host_vals = arr[:nv * 4].view(np.float32)
        # ranges shrinking 4:3:2:1, so the one copy left after the last range
        # is a tenth of the values
        w = np.cumsum([0, 4, 3, 2, 1])
        bounds = [int(nl * int(x) // int(w[-1])) for x in w]
        counts = []
        clip = self.meta.grid_class == "sdf"
        for l0, l1 in zip(bounds[:-1], bounds[1:]):
            if l1 == l0:
                continue
            v0, v1 = l0 * LEAF_SIZE, l1 * LEAF_SIZE
            ids, cnt = self.select(act[v0:v1], 1, sync=False)
            vals = torch.empty(v1 - v0, dtype=torch.float32, device=dev)
            self.evaluate("voxel", _lib.SRC_LEAF_VOX, leaf_origins[l0:l1], v1 - v0, _lib.OUT_VALUE, gather=ids,
                          f32=vals, value_scale=self.value_scale, clip=clip, count=cnt)
            check(lib().nvdb_scatter_f32_unpatched_counted(_ptr(values, 4 * v0), _ptr(ids), _ptr(vals), v1 - v0,
                                                           _ptr(cnt), _ptr(patched, v0), st),
                  "nvdb_scatter_f32_unpatched_counted")
            counts.append(cnt)
            ev = torch.cuda.Event()
            ev.record(torch.cuda.current_stream(dev))
            cs.wait_event(ev)
            with torch.cuda.stream(cs):
                pin[4 * v0:4 * v1].view(torch.float32).copy_(values[v0:v1], non_blocking=True)
        values.record_stream(cs)
        done = torch.cuda.Event()
        done.record(cs)
        acnt = torch.stack(counts).sum(0) if counts else torch.zeros(1, dtype=torch.int64, device=dev)
        d = DeviceDecode(self, cls[:self.n1 * L1_SIZE], tiles[:self.n1 * L1_SIZE], child, leaf_origins[:nl],
                         act[:nv], values, words, patched, acnt, shard, err)
        d.host_vals = ([host_vals], done)
        return d

    def _side_stream(self) -> torch.cuda.Stream:
        """The device's side stream, shared by every DeviceModel: torch's
        caching allocator keeps a block pool per stream, so a new stream per
        model would cudaMalloc the side-stream tables afresh on every
        decode_full call (2 cudaMallocs per call, 3.3 -> 4-110 ms when the
        allocator has no large free block to split)."""
        key = self.dev.index if self.dev.index is not None else torch.cuda.current_device()
        st = _SIDE_STREAMS.get(key)
        if st is None:
            st = _SIDE_STREAMS[key] = torch.cuda.Stream(device=self.dev)
        return st

    def _host_prefetch(self, ts):
        """Asynchronous copies of finished device arrays into one pooled pinned
        block on a side stream, ordered after the work enqueued so far; returns
        (numpy views, completion event)."""
        dev = self.dev
        cs = self._side_stream()
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream(dev))
        cs.wait_event(ev)
        offs, n = [], 0
        for t in ts:
            offs.append(n)
            n += (t.numel() * t.element_size() + 255) & ~255
        pin, arr = _PINNED.get(n)
        outs = []
        with torch.cuda.stream(cs):
            for t, o in zip(ts, offs):
                nb = t.numel() * t.element_size()
                pin[o:o + nb].view(t.dtype).view(t.shape).copy_(t, non_blocking=True)
                outs.append(arr[o:o + nb].view(_NP_DTYPE[t.dtype]).reshape(tuple(t.shape)))
                t.record_stream(cs)
        done = torch.cuda.Event()
        done.record(cs)
        return outs, done


@dataclass
class DeviceDecode:
    """Dense-leaf decode output, resident on the device."""

    model: DeviceModel
    l1_class: torch.Tensor      # (n1*4096,) u8, sorted-origin node order
    l1_tiles: torch.Tensor      # (n1*4096,) f32
    child_slots: torch.Tensor   # (nl,) int64 node*4096 + slot
    leaf_origins: torch.Tensor  # (nl,3) int32
    leaf_active: torch.Tensor   # (nl*512,) u8
    leaf_values: torch.Tensor   # (nl*512,) f32
    active_words: torch.Tensor  # (nl*8,) packed masks (int64 view of u64)
    patched: torch.Tensor       # (nl*512,) u8
    evals_dev: torch.Tensor     # (1,) int64: voxel-regressor evaluations (device)
    shard: Optional[Tuple[int, int]] = None  # (rank, world) when only a leaf range was decoded
    err_dev: Optional[torch.Tensor] = None   # (1,) int32: a level-0 patch fell outside every leaf
    _checked: bool = False
    host_pre: Optional[tuple] = None  # decode(prefetch_host=True): (host arrays, event) of cls / tiles / origins / active / error flags
    host_vals: Optional[tuple] = None  # decode(prefetch_host=True): ([host leaf values], event)

    @property
    def leaf_count(self) -> int:
        return int(self.leaf_origins.shape[0])

    @property
    def regressor_evaluations(self) -> int:
        return int(self.evals_dev.item())

    def check(self) -> "DeviceDecode":
        """Raise SvcodecError for a corrupt container (decoder.py:172-175).  The
        flag is read lazily (first host access) so a decode enqueues without a
        stream synchronisation."""
        if not self._checked and self.err_dev is not None:
            if self.host_pre is not None:  # flags copied to the host with the level-1 / leaf arrays
                (_, _, _, _, e0, e1), done = self.host_pre
                done.synchronize()
                e1, e0 = int(e1[0]), int(e0[0])
            else:
                e1, e0 = int(self.model.err[0].item()), int(self.err_dev.item())
            if e1:  # decoder.py:121-124
                raise SvcodecError("corrupt container: level-1 patch outside every level-1 node")
            if e0:
                raise SvcodecError("corrupt container: level-0 patch outside every reconstructed leaf")
            self._checked = True
        return self

    def to_grid(self) -> DenseLeafGrid:
        """Host DenseLeafGrid in canonical (root, idx2, idx1) order."""
        if self.shard is not None and self.shard[1] > 1:
            raise ValueError("a sharded decode holds a leaf range, not a grid; gather the shards first")
        self.check()
        m = self.model
        c = m.c
        meta = c.grid_meta
        bg = np.float32(meta.background)
        n1 = m.n1
        vdone = None
        if self.host_pre is not None:
            (cls, tiles, lo, la, _, _), done = self.host_pre
            if self.host_vals is not None:
                (lv,), vdone = self.host_vals  # waited for below, after the host-side ordering
            else:
                (lv,) = _to_host([self.leaf_values])
            done.synchronize()
        else:
            cls, tiles, lo, la, lv = _to_host([self.l1_class, self.l1_tiles, self.leaf_origins,
                                               self.leaf_active, self.leaf_values])
        cls = cls.reshape(n1, L1_SIZE)
        tiles = tiles.reshape(n1, L1_SIZE)
        lo = lo.astype(np.int64).reshape(-1, 3)
        la = la.view(np.bool_).reshape(-1, LEAF_SIZE)  # 0/1 bytes
        lv = lv.reshape(-1, LEAF_SIZE)
        # canonical order: by root key then origin within the root
        roots = m.origins & ~np.int64(4095)
        order = np.lexsort((m.origins[:, 2], m.origins[:, 1], m.origins[:, 0],
                            roots[:, 2], roots[:, 1], roots[:, 0])) if n1 else np.zeros(0, np.int64)
        counts = (cls == 0).sum(axis=1)
        starts = np.concatenate([[0], np.cumsum(counts)[:-1]]) if n1 else np.zeros(0, np.int64)
        leaf_perm = np.concatenate([np.arange(starts[i], starts[i] + counts[i]) for i in order]) \
            if n1 else np.zeros(0, np.int64)
        leaf_perm = leaf_perm.astype(np.int64)
        ident = leaf_perm.shape[0] == lo.shape[0] and bool(np.array_equal(leaf_perm, np.arange(lo.shape[0])))
        ut = c.upper_tree
        l2o = np.asarray([n.origin for n in ut.l2_nodes], dtype=np.int64).reshape(-1, 3)
        o2 = np.lexsort((l2o[:, 2], l2o[:, 1], l2o[:, 0])) if len(l2o) else np.zeros(0, np.int64)
        l2c = np.zeros((len(o2), L2_SIZE), bool)
        l2a = np.zeros((len(o2), L2_SIZE), bool)
        l2t = np.full((len(o2), L2_SIZE), bg, np.float32)
        for j, i in enumerate(o2):
            nd = ut.l2_nodes[i]
            l2c[j] = nd.child_mask.bits
            l2a[j] = nd.active_mask.bits
            for k, v in nd.tiles.items():
                l2t[j, int(k)] = v
        if vdone is not None:
            vdone.synchronize()
        return DenseLeafGrid(
            background=float(meta.background), grid_class=meta.grid_class, voxel_size=float(meta.voxel_size),
            half_width=float(meta.half_width), root_tiles=dict(ut.root_tiles),
            l2_origins=l2o[o2], l2_child=l2c, l2_active=l2a, l2_tiles=l2t,
            l1_origins=m.origins[order], l1_child=(cls == 0)[order], l1_active=(cls == 1)[order],
            l1_tiles=tiles[order], leaf_origins=lo if ident else lo[leaf_perm],
            leaf_active=la if ident else la[leaf_perm], leaf_values=lv if ident else lv[leaf_perm])

    def to_nvgr(self) -> bytes:
        """The decoded grid as NVGR bytes, identical to
        ``gridfile.serialize_grid(decode_full(c))`` (gridfile.py:43-76).

        The level-1 node and leaf records -- all but a few hundred bytes per
        root entry -- are written on the device straight from the dense-leaf
        output (``nvdb_nvgr_l1_records`` / ``nvdb_nvgr_leaf_records``) and come
        back in one copy; the host adds the header, the root entries and the
        level-2 node blocks from the container's upper tree."""
        import struct
        if self.shard is not None and self.shard[1] > 1:
            raise ValueError("a sharded decode holds a leaf range, not a grid; gather the shards first")
        self.check()
        m = self.model
        c = m.c
        meta = c.grid_meta
        ut = c.upper_tree
        n1, dev = m.n1, m.dev
        bg = np.float32(meta.background)
        L2REC, L1REC, LEAFREC = 4096 + 4096 + 4 * L2_SIZE, 12 + 512 + 512 + 4 * L1_SIZE, 12 + 64 + 4 * LEAF_SIZE
        cnt = (self.l1_class.view(max(n1, 0), L1_SIZE) == 0).sum(dim=1) if n1 else torch.zeros(0, device=dev)
        cnt = cnt.to(torch.int64).cpu().numpy()
        org = m.origins  # decode node order (sorted origins)
        roots = org & ~np.int64(4095)
        l2 = {tuple(int(v) for v in nd.origin): nd for nd in ut.l2_nodes}
        keys = sorted(set(l2) | set(ut.root_tiles))
        # level-1 nodes per root in NVGR order (ascending idx2 == ascending origin in a root)
        by_root: Dict[tuple, list] = {}
        for i, r in enumerate(map(tuple, roots.tolist())):
            by_root.setdefault(r, []).append(i)
        off = 4 + 4 + 1 + 4 + 8 + 4 + 8
        l1_off = np.zeros(n1, np.int64)
        host_parts = []  # (offset, bytes)
        header = b"NVGR" + struct.pack("<IBfdfQ", 1, 0 if meta.grid_class == "sdf" else 1, float(bg),
                                       float(meta.voxel_size), float(np.float32(meta.half_width)), len(keys))
        host_parts.append((0, header))
        for key in keys:
            tile = ut.root_tiles.get(key)
            if tile is not None:
                host_parts.append((off, struct.pack("<iiiBfB", *key, 1, float(tile[0]), int(bool(tile[1])))))
                off += 13 + 5
                continue
            nd = l2[key]
            tiles = np.full(L2_SIZE, bg, np.float32)
            if nd.tiles:
                tiles[np.fromiter(nd.tiles.keys(), np.int64, len(nd.tiles))] = np.fromiter(
                    nd.tiles.values(), np.float32, len(nd.tiles))
            blob = (struct.pack("<iiiB", *key, 0)
                    + np.packbits(np.asarray(nd.child_mask.bits, bool), bitorder="little").tobytes()
                    + np.packbits(np.asarray(nd.active_mask.bits, bool), bitorder="little").tobytes()
                    + tiles.tobytes())
            host_parts.append((off, blob))
            off += 13 + L2REC
            mine = by_root.get(key, [])
            if mine:
                sizes = L1REC + cnt[mine] * LEAFREC
                l1_off[mine] = off + np.concatenate([[0], np.cumsum(sizes)[:-1]])
                off += int(sizes.sum())
        total = off
        out = torch.empty(max(total, 1), dtype=torch.uint8, device=dev)
        st = _stream(dev)
        nl = self.leaf_count
        if n1:
            d_l1 = torch.from_numpy(l1_off).to(dev)
            check(lib().nvdb_nvgr_l1_records(_ptr(m.d_origins), _ptr(self.l1_class), _ptr(self.l1_tiles), n1,
                                             _ptr(d_l1), _ptr(out), st), "nvdb_nvgr_l1_records")
        if nl:
            # leaf j of node i (decode order, node-contiguous): l1_off[i] + L1REC + (j - first_i) * LEAFREC
            node = torch.repeat_interleave(torch.arange(n1, device=dev), torch.from_numpy(cnt).to(dev))
            first = torch.from_numpy(np.concatenate([[0], np.cumsum(cnt)[:-1]]).astype(np.int64)).to(dev)
            j = torch.arange(nl, device=dev)
            leaf_off = d_l1[node] + L1REC + (j - first[node]) * LEAFREC
            check(lib().nvdb_nvgr_leaf_records(_ptr(self.leaf_origins), _ptr(self.active_words),
                                               _ptr(self.leaf_values), nl, _ptr(leaf_off), _ptr(out), st),
                  "nvdb_nvgr_leaf_records")
        (host,) = _to_host([out[:total]])
        buf = bytearray(host.tobytes())
        for o, b in host_parts:
            buf[o:o + len(b)] = b
        return bytes(buf)

    def tree(self) -> DeviceTree:
        """Device tree over this decode (hybrid topology for random access)."""
        return DeviceTree.from_decode(self)


def shard_range(nleaves: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous leaf range of one decode shard (split the
    node-ordered leaf list into equal ranges; no collective)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad shard {rank}/{world}")
    return nleaves * rank // world, nleaves * (rank + 1) // world


def gather_rows(parts, group=None, dst: int = 0):
    """Concatenate every rank's row blocks, in rank order, on rank ``dst``.

    ``parts``: this rank's tensors, each (n_rank, ...) with the same row count
    n_rank across the list (row counts may differ between ranks).  One
    all-gather of the counts, then one all-gather per tensor of the blocks
    padded to the largest count (NCCL over NVLink for device tensors, gloo for
    host tensors).  Returns the concatenated tensors on ``dst`` and None
    elsewhere.  SURVEY.md §8(e): the optional gather of dense-leaf outputs."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    dev = parts[0].device
    n = int(parts[0].shape[0])
    cnt = torch.tensor([n], dtype=torch.int64, device=dev)
    allc = [torch.zeros_like(cnt) for _ in range(world)]
    dist.all_gather(allc, cnt, group=group)
    counts = [int(c.item()) for c in allc]
    mx = max(max(counts), 1)
    out = []
    for t in parts:
        pad = torch.zeros((mx,) + tuple(t.shape[1:]), dtype=t.dtype, device=dev)
        pad[:n] = t[:n]
        bufs = [torch.empty_like(pad) for _ in range(world)]
        dist.all_gather(bufs, pad, group=group)
        out.append(torch.cat([b[:c] for b, c in zip(bufs, counts)]) if rank == dst else None)
    return out if rank == dst else None


def _as_model(c, device=None) -> DeviceModel:
    return c if isinstance(c, DeviceModel) else DeviceModel(c, device)


def decode_nvgr(c, device=None, group=None) -> Optional[bytes]:
    """``gridfile.serialize_grid(decoder.decode_full(c))`` (decoder.py:214,
    gridfile.py:43-76) with the records emitted on the device: the decoded
    grid as NVGR bytes, no per-node host objects.  With a process group the
    decode is sharded and rank 0 returns the bytes (None elsewhere)."""
    m = _as_model(c, device)
    if group is not None and _world(group) > 1:
        d = decode_sharded(m, group)
        if d is None:
            return None
    else:
        d = m.decode(True)
    return d.to_nvgr()


def decode_sharded(m: DeviceModel, group=None, dst: int = 0) -> Optional["DeviceDecode"]:
    """Decode over the ranks of ``group`` (one process per GPU): every rank
    classifies the level-1 slots (cheap, redundant), decodes its contiguous
    leaf range, and the dense-leaf blocks are gathered in leaf order on rank
    ``dst`` (PAPER.md:253 disjoint-block decode).  Returns
    the full DeviceDecode on ``dst``, None elsewhere."""
    import torch.distributed as dist
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    d = m.decode(True, shard=(rank, world)).check()
    nl = d.leaf_count
    parts = [d.child_slots[:nl], d.leaf_origins[:nl], d.leaf_active.view(nl, LEAF_SIZE),
             d.leaf_values.view(nl, LEAF_SIZE), d.active_words.view(nl, 8), d.patched.view(nl, LEAF_SIZE)]
    g = gather_rows(parts, group, dst)
    ev = torch.zeros(1, dtype=torch.int64, device=m.dev)
    ev += d.evals_dev
    dist.all_reduce(ev, group=group)
    if g is None:
        return None
    child, lo, la, lv, w, pt = g
    return DeviceDecode(m, d.l1_class, d.l1_tiles, child, lo, la.reshape(-1), lv.reshape(-1), w.reshape(-1),
                        pt.reshape(-1), ev, None, None, True)


def decode_full(c, device=None, as_svcodec: bool = False, group=None):
    """decoder.decode_full (decoder.py:214-217): the complete explicit grid.

    Returns a :class:`DenseLeafGrid` (or an svcodec ``VdbGrid`` with
    ``as_svcodec=True`` when the reference package is importable).  With a
    ``torch.distributed`` group of G > 1 ranks (one per GPU) the leaves are
    decoded in G contiguous ranges and gathered on rank 0, which returns the
    grid; the other ranks return None.
    """
    m = _as_model(c, device)
    if group is not None and _world(group) > 1:
        d = decode_sharded(m, group)
        if d is None:
            return None
    else:
        d = m.decode(True, prefetch_host=True)
    g = d.to_grid()
    return g.to_svcodec() if as_svcodec else g


def _world(group) -> int:
    import torch.distributed as dist
    return dist.get_world_size(group)


def decode_report(c, device=None) -> Dict[str, int]:
    """decoder.decode_report (decoder.py:294-300)."""
    m = _as_model(c, device)
    d = m.decode(True).check()
    return {"regressor_evaluations": d.regressor_evaluations,
            "active_voxels": int(d.leaf_active.sum().item())}


def hybrid_query(tree: DeviceTree, nets, coords: torch.Tensor, value_scale: float, clip: bool):
    """Explicit-topology lookup + neural values on active leaf voxels
    (decoder.py:239-264): K1 lookup, select the rows that resolve to an
    active leaf voxel, gate-blended voxel regressor on exactly those rows,
    scatter.  ``nets`` is a DeviceModel or NetEvaluator.  Returns (values,
    active, regressor evaluations)."""
    dev, st = nets.dev, _stream(nets.dev)
    n = coords.shape[0]
    # one pass: lookup + the active leaf-voxel rows (patched rows keep their
    # exact value and only count as evaluated, as the reference's finalize)
    val, act, kind, rows, cnt, npatched = tree.lookup_rows(coords)
    if n:
        reg = torch.empty(max(n, 1), dtype=torch.float32, device=dev)
        nets.evaluate("voxel", _lib.SRC_COORD_I32, coords, n, _lib.OUT_VALUE, gather=rows, f32=reg,
                      value_scale=value_scale, clip=clip, count=cnt)
        check(lib().nvdb_scatter_f32_counted(_ptr(val), _ptr(rows), _ptr(reg), n, _ptr(cnt), st),
              "nvdb_scatter_f32_counted")
    return val, act, cnt + npatched


class HybridGrid:
    """Explicit topology with neural leaf values (decoder.py:222-264)."""

    def __init__(self, model: DeviceModel, topo: DeviceDecode):
        self.model = model
        self.container = model.c
        self.topology_decode = topo
        self.tree = topo.tree()
        self.regressor_evaluations = 0

    @property
    def topology(self) -> DenseLeafGrid:
        return self.topology_decode.to_grid()

    def query_device(self, coords: torch.Tensor):
        """(values f32, active u8) for device int32 coords (n,3)."""
        m = self.model
        val, act, nr = hybrid_query(self.tree, m, coords, m.value_scale, m.meta.grid_class == "sdf")
        self._evals.append(nr)
        return val, act

    @property
    def regressor_evaluations(self) -> int:
        """Voxel-regressor rows over all queries so far (decoder.py:262-263)."""
        if self._evals:
            self._base += int(sum(int(t.item()) for t in self._evals))
            self._evals = []
        return self._base

    @regressor_evaluations.setter
    def regressor_evaluations(self, v: int) -> None:
        self._evals, self._base = [], int(v)

    def query(self, coords, group=None) -> Tuple[np.ndarray, np.ndarray]:
        """Batched (value, active) at integer coordinates (decoder.py:239-264).

        With a ``torch.distributed`` group of G > 1 ranks every rank passes the
        same coordinates, queries its contiguous 1/G slice on its own GPU (tree
        and nets replicated, no collective on the data path), and rank 0
        returns all results in order (gathered over NCCL); other ranks return
        (None, None).  SURVEY.md §8(e) "Random query"."""
        c = np.asarray(coords)
        lim = 1 << 30
        if c.dtype != np.int32:
            c = c.astype(np.int64).reshape(-1, 3)
            if c.size and (c.max() >= lim or c.min() <= -lim):  # grid.py:69-71
                raise SvcodecError("coordinate outside legal range +-2^30")
            c = c.astype(np.int32)
        c = c.reshape(-1, 3)
        if group is not None and _world(group) > 1:
            import torch.distributed as dist
            lo, hi = shard_range(c.shape[0], dist.get_rank(group), _world(group))
            c = c[lo:hi]
        d = _to_device(c, self.model.dev)
        # int32 input: the +-2^30 range check runs on the device, read with the results
        bad = ((d >= lim) | (d <= -lim)).any().view(1).to(torch.uint8)
        v, a = self.query_device(d)
        if group is not None and _world(group) > 1:
            import torch.distributed as dist
            bad32 = bad.to(torch.int32)
            dist.all_reduce(bad32, op=dist.ReduceOp.MAX, group=group)
            g = gather_rows([v, a], group)
            if g is None:
                return None, None
            v, a = g
            bad = bad32.to(torch.uint8)
        v, a, bad = _to_host([v, a, bad])
        if bad.any():
            raise SvcodecError("coordinate outside legal range +-2^30")
        # views of a pooled pinned block (free again once the caller drops them)
        return v, a.view(np.bool_)


def make_hybrid(c, device=None) -> HybridGrid:
    """decoder.make_hybrid (decoder.py:267-270)."""
    m = _as_model(c, device)
    return HybridGrid(m, m.decode(False))
