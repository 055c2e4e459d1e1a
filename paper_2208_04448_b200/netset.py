"""Device netset: every expert's networks uploaded once for the CUDA kernels.

Replaces the per-call net handling of ``inference.eval_net``
(inference.py:23-26): weights are packed (fp16, UMMA layout, omega and
amplitude folded) by ``nvdb_netset_create`` and stay resident.
"""

from __future__ import annotations

import ctypes as C
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np
import torch

from . import _lib
from ._lib import ExpertDesc, NetDesc, check, lib

ACT_CODES = {"relu": 0, "tanh": 1, "sine": 2}
HEAD_CODES = {"linear": 0, "logits": 1, "binary": 2}
TAGS = ("l1", "tile", "l0", "voxel")
TAG_CODES = {t: i for i, t in enumerate(TAGS)}


def b2pi_f32(ff) -> np.ndarray:
    """(2*pi*B^T) rounded to float32 exactly as neural.py:421/537 does."""
    return np.ascontiguousarray((2.0 * np.pi * np.asarray(ff.matrix).T).astype(np.float32))


def _net_desc(params, ff, keep: list) -> NetDesc:
    layers = params.layers
    depth = len(layers) - 1
    # unequal hidden widths are zero-padded to the widest layer: padded units
    # see zero weights and bias, act(0) = 0 for relu/tanh/sine, so the padded
    # net computes the same function
    width = max(w.shape[0] for w, _ in layers[:-1])
    ws, bs = [], []
    for li, (w, b) in enumerate(layers):
        w = np.asarray(w, dtype=np.float32)
        b = np.asarray(b, dtype=np.float32)
        rows = w.shape[0] if li == depth else width
        cols = w.shape[1] if li == 0 else width
        wp = np.zeros((rows, cols), dtype=np.float32)
        wp[:w.shape[0], :w.shape[1]] = w
        bp = np.zeros(rows, dtype=np.float32)
        bp[:b.shape[0]] = b
        ws.append(np.ascontiguousarray(wp))
        bs.append(bp)
    if ws[0].shape[1] != 2 * ff.m:
        raise ValueError(f"first layer expects {ws[0].shape[1]} inputs, features give {2 * ff.m}")
    b2 = b2pi_f32(ff)
    wp = (C.POINTER(C.c_float) * len(ws))(*[w.ctypes.data_as(C.POINTER(C.c_float)) for w in ws])
    bp = (C.POINTER(C.c_float) * len(bs))(*[b.ctypes.data_as(C.POINTER(C.c_float)) for b in bs])
    keep.extend([ws, bs, b2, wp, bp])
    return NetDesc(m=ff.m, depth=depth, width=width, out_dim=ws[-1].shape[0],
                   activation=ACT_CODES[params.activation.kind], head=HEAD_CODES[params.head],
                   frequency=float(params.activation.frequency), amplitude=float(ff.amplitude),
                   b2pi=b2.ctypes.data_as(C.POINTER(C.c_float)), weights=wp, biases=bp)


class DeviceNetSet:
    """All experts' nets on the current CUDA device.

    ``experts`` must be in subdomain-id order (ascending cells), as produced
    by ``decompose`` (partition.py:90-94).
    """

    def __init__(self, experts: Sequence, subdomain_size: int, halo: int = 8, device=None):
        descs: List[NetDesc] = []
        exps: List[ExpertDesc] = []
        keep: list = []
        self.net_of: Dict[Tuple[int, str], int] = {}
        self.out_dims: List[int] = []
        for ei, e in enumerate(experts):
            idx = [-1, -1, -1, -1]
            for tag, rec in e.nets():
                if rec is None:
                    continue
                idx[TAG_CODES[tag]] = len(descs)
                self.net_of[(ei, tag)] = len(descs)
                descs.append(_net_desc(rec.params, rec.ff, keep))
                self.out_dims.append(rec.params.layers[-1][0].shape[0])
            no = np.asarray(e.norm_origin, dtype=np.float64)
            exps.append(ExpertDesc(cell=(C.c_int32 * 3)(*[int(v) for v in e.cell]),
                                   net_index=(C.c_int32 * 4)(*idx),
                                   norm_origin=(C.c_double * 3)(*[float(v) for v in no]),
                                   norm_scale=float(e.norm_scale)))
        darr = (NetDesc * max(len(descs), 1))(*descs)
        earr = (ExpertDesc * max(len(exps), 1))(*exps)
        handle = C.c_void_p()
        # device memory from the caller (torch's caching allocator) and an
        # upload ordered on the current stream: no cudaMalloc / cudaFree and no
        # host synchronisation per net set (nvdb_netset_create_at)
        need = C.c_size_t()
        check(lib().nvdb_netset_device_bytes(darr, len(descs), earr, len(exps), int(subdomain_size), int(halo),
                                             C.byref(need)), "nvdb_netset_device_bytes")
        dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        self.mem = torch.empty(int(need.value), dtype=torch.uint8, device=dev)
        check(lib().nvdb_netset_create_at(darr, len(descs), earr, len(exps), int(subdomain_size), int(halo),
                                          self.mem.data_ptr(), self.mem.numel(),
                                          torch.cuda.current_stream(dev).cuda_stream, C.byref(handle)),
              "nvdb_netset_create_at")
        self.handle = handle
        self.nexperts = len(exps)

    def close(self) -> None:
        if getattr(self, "handle", None) is not None and self.handle.value:
            lib().nvdb_netset_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass

    # -- kernels -------------------------------------------------------------

    def forward(self, net: int, pts: torch.Tensor, out: Optional[torch.Tensor] = None) -> torch.Tensor:
        """Raw outputs of one net at normalized points (forward_block seam)."""
        assert pts.is_cuda and pts.dtype == torch.float32 and pts.is_contiguous()
        n = pts.shape[0]
        od = self.out_dims[net]
        if out is None:
            out = torch.empty((n, od), dtype=torch.float32, device=pts.device)
        stream = torch.cuda.current_stream(pts.device).cuda_stream
        check(lib().nvdb_forward(self.handle, net, pts.data_ptr(), n, out.data_ptr(), stream), "nvdb_forward")
        return out

    def blended(self, tag: str, centers: torch.Tensor):
        """Gate-blended (n,k) f64 outputs + covered u8 at f64 centres."""
        assert centers.is_cuda and centers.dtype == torch.float64 and centers.is_contiguous()
        n = centers.shape[0]
        k = 3 if tag == "l1" else 1
        out = torch.empty((n, k), dtype=torch.float64, device=centers.device)
        cov = torch.empty((n,), dtype=torch.uint8, device=centers.device)
        wsb = lib().nvdb_eval_workspace_bytes(self.handle, n)
        ws = torch.empty((max(int(wsb), 1),), dtype=torch.uint8, device=centers.device)
        stream = torch.cuda.current_stream(centers.device).cuda_stream
        check(lib().nvdb_eval_blended(self.handle, TAG_CODES[tag], centers.data_ptr(), n, out.data_ptr(),
                                      cov.data_ptr(), ws.data_ptr(), ws.numel(), stream), "nvdb_eval_blended")
        return out, cov
