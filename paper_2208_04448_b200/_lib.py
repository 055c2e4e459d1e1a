"""ctypes binding of the C ABI in ``include/nvdb_b200.h``.

The shared library is built in-tree (``csrc/Makefile`` -> ``libnvdb_b200.so``
next to this file).  There is no CPU fallback: if the library or a CUDA
device is missing, every compute entry point raises.
"""

from __future__ import annotations

import ctypes as C
import os
from typing import Optional

from .errors import SvcodecError

HERE = os.path.dirname(os.path.abspath(__file__))
# NVDB_LIB selects a debug build (e.g. libnvdb_b200_trace.so) for diagnostics
LIB_PATH = os.path.join(HERE, os.environ.get("NVDB_LIB", "libnvdb_b200.so"))

NVDB_OK = 0
NVDB_EINVAL = -1
NVDB_ECUDA = -2
NVDB_EUNSUPPORTED = -3
NVDB_ECORRUPT = -4
NVDB_ENOMEM = -5

EXPORTED = [
    "nvdb_last_error", "nvdb_version", "nvdb_launch_count", "nvdb_netset_create", "nvdb_netset_destroy",
    "nvdb_forward", "nvdb_eval_workspace_bytes", "nvdb_eval_blended", "nvdb_tree_create",
    "nvdb_tree_destroy", "nvdb_lookup", "nvdb_lookup_rows", "nvdb_selftest_umma", "nvdb_eval",
    "nvdb_select_workspace_bytes", "nvdb_select_u8", "nvdb_l1_apply", "nvdb_scatter_f32",
    "nvdb_leaf_list", "nvdb_l0_apply", "nvdb_leaf_finalize", "nvdb_pack_eq", "nvdb_neural_rows",
    "nvdb_query_finalize", "nvdb_trainer_create", "nvdb_trainer_destroy", "nvdb_trainer_run",
    "nvdb_trainer_status", "nvdb_trainer_weights", "nvdb_sample_indices", "nvdb_trainer_phase",
    "nvdb_trainer_buffers", "nvdb_sample_indices_subset", "nvdb_fbm_leaves", "nvdb_trim",
    "nvdb_eval_counted", "nvdb_leaf_finalize_counted", "nvdb_scatter_f32_counted", "nvdb_scatter_f32_unpatched_counted",
    "nvdb_query_finalize_counted", "nvdb_trainer_packed", "nvdb_nvgr_leaf_records", "nvdb_nvgr_l1_records",
    "nvdb_metric_partials", "nvdb_metric_pass", "nvdb_trainer_set_ctas", "nvdb_netset_device_bytes",
    "nvdb_netset_create_at", "nvdb_node_slots",
]

SRC_NORM_F32, SRC_CENTER_F64, SRC_COORD_I32, SRC_LEAF_VOX, SRC_L1_SLOT = range(5)
OUT_RAW, OUT_PROBS, OUT_L1CLASS, OUT_L0ACTIVE, OUT_VALUE = range(5)


class EvalOut(C.Structure):
    _fields_ = [("out_mode", C.c_int32), ("raw", C.c_void_p), ("probs", C.c_void_p),
                ("u8", C.c_void_p), ("f32", C.c_void_p), ("value_scale", C.c_double),
                ("background", C.c_float), ("clip", C.c_int32)]


class NetDesc(C.Structure):
    _fields_ = [("m", C.c_int32), ("depth", C.c_int32), ("width", C.c_int32),
                ("out_dim", C.c_int32), ("activation", C.c_int32), ("head", C.c_int32),
                ("frequency", C.c_float), ("amplitude", C.c_float),
                ("b2pi", C.POINTER(C.c_float)),
                ("weights", C.POINTER(C.POINTER(C.c_float))),
                ("biases", C.POINTER(C.POINTER(C.c_float)))]


class ExpertDesc(C.Structure):
    _fields_ = [("cell", C.c_int32 * 3), ("net_index", C.c_int32 * 4),
                ("norm_origin", C.c_double * 3), ("norm_scale", C.c_double)]


class TreeDesc(C.Structure):
    _fields_ = [("background", C.c_float), ("nroots", C.c_int32), ("n2", C.c_int32),
                ("n1", C.c_int32), ("nl", C.c_int32),
                ("root_keys", C.c_void_p), ("root_l2", C.c_void_p),
                ("root_tile_value", C.c_void_p), ("root_tile_active", C.c_void_p),
                ("l2_child", C.c_void_p), ("l2_active", C.c_void_p), ("l2_tiles", C.c_void_p),
                ("l2_child_base", C.c_void_p), ("l1_child", C.c_void_p), ("l1_active", C.c_void_p),
                ("l1_tiles", C.c_void_p), ("l1_child_base", C.c_void_p),
                ("leaf_active", C.c_void_p), ("leaf_values", C.c_void_p),
                ("leaf_patched", C.c_void_p)]


class TrainDesc(C.Structure):
    _fields_ = [("net", NetDesc), ("loss_kind", C.c_int32), ("n", C.c_int64), ("inputs", C.c_void_p),
                ("targets", C.c_void_p), ("batch", C.c_int32), ("sampled", C.c_int32),
                ("sample_interval", C.c_int32), ("max_epochs", C.c_int32), ("lr", C.c_void_p),
                ("c1", C.c_void_p), ("c2", C.c_void_p), ("seed_words", C.c_void_p),
                ("target_loss", C.c_double), ("shard_rank", C.c_int32), ("shard_count", C.c_int32),
                ("path", C.c_int32)]


class FbmDesc(C.Structure):
    _fields_ = [("octaves", C.c_int32), ("lacunarity", C.c_double), ("gain", C.c_double),
                ("base_frequency", C.c_double), ("seed", C.c_uint64), ("lo", C.c_int32 * 3),
                ("hi", C.c_int32 * 3), ("threshold", C.c_double), ("voxel_size", C.c_double)]


_lib: Optional[C.CDLL] = None


def _declare(lib: C.CDLL) -> None:
    vp, i32, i64, u32, sz = C.c_void_p, C.c_int32, C.c_int64, C.c_uint32, C.c_size_t
    sig = {
        "nvdb_last_error": (C.c_char_p, []),
        "nvdb_version": (C.c_int, []),
        "nvdb_launch_count": (C.c_longlong, []),
        "nvdb_netset_create": (C.c_int, [C.POINTER(NetDesc), i32, C.POINTER(ExpertDesc), i32, i32, i32,
                                         C.POINTER(vp)]),
        "nvdb_netset_destroy": (C.c_int, [vp]),
        "nvdb_netset_device_bytes": (C.c_int, [C.POINTER(NetDesc), i32, C.POINTER(ExpertDesc), i32, i32, i32,
                                               C.POINTER(sz)]),
        "nvdb_netset_create_at": (C.c_int, [C.POINTER(NetDesc), i32, C.POINTER(ExpertDesc), i32, i32, i32, vp, sz,
                                            vp, C.POINTER(vp)]),
        "nvdb_forward": (C.c_int, [vp, i32, vp, i64, vp, vp]),
        "nvdb_eval_workspace_bytes": (sz, [vp, i64]),
        "nvdb_eval_blended": (C.c_int, [vp, i32, vp, i64, vp, vp, vp, sz, vp]),
        "nvdb_tree_create": (C.c_int, [C.POINTER(TreeDesc), C.POINTER(vp)]),
        "nvdb_tree_destroy": (C.c_int, [vp]),
        "nvdb_lookup": (C.c_int, [vp, vp, i64, vp, vp, vp, vp, vp]),
        "nvdb_lookup_rows": (C.c_int, [vp, vp, i64, vp, vp, vp, vp, vp, vp, vp]),
        "nvdb_selftest_umma": (C.c_int, [vp, u32, vp, u32, i32, i32, u32, u32, u32, u32, u32, u32,
                                         i32, i32, vp, vp]),
        "nvdb_eval": (C.c_int, [vp, i32, i32, vp, vp, i64, C.POINTER(EvalOut), vp, sz, vp]),
        "nvdb_eval_counted": (C.c_int, [vp, i32, i32, vp, vp, i64, vp, C.POINTER(EvalOut), vp, sz, vp]),
        "nvdb_select_workspace_bytes": (sz, [i64]),
        "nvdb_select_u8": (C.c_int, [vp, i64, C.c_uint8, vp, vp, vp, sz, vp]),
        "nvdb_l1_apply": (C.c_int, [vp, vp, i64, vp, vp, i64, vp, vp, i64, vp]),
        "nvdb_scatter_f32": (C.c_int, [vp, vp, vp, i64, vp]),
        "nvdb_leaf_list": (C.c_int, [vp, i64, vp, i64, vp, vp, vp]),
        "nvdb_node_slots": (C.c_int, [vp, C.POINTER(i32), C.POINTER(i32), vp, i64, vp, vp, vp, vp]),
        "nvdb_l0_apply": (C.c_int, [vp, vp, vp, vp, i64, vp, vp, vp]),
        "nvdb_leaf_finalize": (C.c_int, [i64, vp, vp, vp, i64, vp, vp, vp, vp, i64, vp, vp, i64, vp,
                                         C.c_float, C.c_float, vp, vp, vp, vp]),
        "nvdb_leaf_finalize_counted": (C.c_int, [i64, vp, vp, vp, i64, vp, vp, vp, vp, vp, i64, vp, vp, i64, vp,
                                                 C.c_float, C.c_float, vp, vp, vp, vp]),
        "nvdb_scatter_f32_counted": (C.c_int, [vp, vp, vp, i64, vp, vp]),
        "nvdb_scatter_f32_unpatched_counted": (C.c_int, [vp, vp, vp, i64, vp, vp, vp]),
        "nvdb_pack_eq": (C.c_int, [vp, i64, C.c_uint8, vp, vp]),
        "nvdb_neural_rows": (C.c_int, [vp, vp, i64, vp, vp]),
        "nvdb_query_finalize": (C.c_int, [vp, i64, vp, vp, vp, vp, vp, vp]),
        "nvdb_query_finalize_counted": (C.c_int, [vp, i64, vp, vp, vp, vp, vp, vp, vp]),
        "nvdb_trainer_create": (C.c_int, [C.POINTER(TrainDesc), C.POINTER(vp)]),
        "nvdb_trainer_destroy": (C.c_int, [vp]),
        "nvdb_trim": (sz, []),
        "nvdb_trainer_run": (C.c_int, [vp, i32, vp]),
        "nvdb_trainer_set_ctas": (C.c_int, [vp, i32]),
        "nvdb_trainer_status": (C.c_int, [vp, C.POINTER(i32), C.POINTER(i32), vp, i32]),
        "nvdb_trainer_weights": (C.c_int, [vp, C.POINTER(C.POINTER(C.c_float)), C.POINTER(C.POINTER(C.c_float))]),
        "nvdb_sample_indices": (C.c_int, [C.c_uint64, i64, vp, vp, vp]),
        "nvdb_sample_indices_subset": (C.c_int, [C.c_uint64, i64, i32, vp, vp, vp, vp]),
        "nvdb_fbm_leaves": (C.c_int, [C.POINTER(FbmDesc), vp, i64, vp, vp, vp, vp]),
        "nvdb_trainer_phase": (C.c_int, [vp, i32, vp]),
        "nvdb_trainer_packed": (C.c_int, [vp, C.POINTER(C.c_void_p), C.POINTER(i64)]),
        "nvdb_nvgr_leaf_records": (C.c_int, [vp, vp, vp, i64, vp, vp, vp]),
        "nvdb_nvgr_l1_records": (C.c_int, [vp, vp, vp, i64, vp, vp, vp]),
        "nvdb_metric_partials": (sz, []),
        "nvdb_metric_pass": (C.c_int, [vp, vp, vp, vp, vp, vp, vp, vp, i64, i32, i32, vp, vp]),
        "nvdb_trainer_buffers": (C.c_int, [vp, C.POINTER(C.c_void_p), C.POINTER(i64), C.POINTER(C.c_void_p)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args


def lib() -> C.CDLL:
    """Load the CUDA library (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `make -C {os.path.join(HERE, 'csrc')}` "
                "(or __graft_entry__.build()); there is no CPU fallback")
        _lib = C.CDLL(LIB_PATH)
        _declare(_lib)
    return _lib


class NvdbError(RuntimeError):
    """CUDA or unsupported-shape failure reported by the C ABI."""


def check(rc: int, what: str = "") -> None:
    if rc == NVDB_OK:
        return
    msg = lib().nvdb_last_error().decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if rc == NVDB_EINVAL:
        raise ValueError(text)
    if rc == NVDB_ECORRUPT:
        raise SvcodecError(text)
    raise NvdbError(f"[{rc}] {text}")
