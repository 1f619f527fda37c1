"""ctypes binding of libjzknn.so (include/jz_knn.h). Argument marshalling only: every
step of the kNN path runs in the library's CUDA kernels. There is no CPU fallback: if the
library is missing or no CUDA device is present, calls raise.
"""
from __future__ import annotations

import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libjzknn.so")

JZ_OK, JZ_EINVAL, JZ_EDATA, JZ_ECAPACITY, JZ_ECUDA, JZ_ENCCL, JZ_ENOMEM = 0, 2, 3, 4, 5, 6, 7
JZ_ORDER_INPUT, JZ_ORDER_Z = 0, 1
JZ_FLAG_FRAME, JZ_FLAG_NO_EARLY_EXIT, JZ_FLAG_NO_SEGSORT, JZ_FLAG_QBOX_DIAG = 1, 2, 4, 8

# every symbol include/jz_knn.h declares (tests check the library exports them all)
EXPORTS = [
    "jz_knn_build", "jz_knn_build_xyzg", "jz_knn_build_xq", "jz_knn_rows", "jz_knn_query", "jz_knn_free", "jz_knn_search_host",
    "jz_knn_stage_times", "jz_set_timing", "jz_last_error", "jz_morton_keys", "jz_bucket_by_splitters",
    "jz_pack_by_rank", "jz_knn_plane_nodes", "jz_knn_query_boxes", "jz_knn_select_ghosts", "jz_knn_pack_ghosts",
    "jz_knn_debug_copy", "jz_launch_count", "jz_knn_stats", "jz_pack_rows", "jz_scatter_rows",
    "jz_fof", "jz_fof_catalogue",
    "jz_comm_unique_id", "jz_comm_init", "jz_comm_local_world", "jz_comm_init_local", "jz_comm_rank_size",
    "jz_comm_free", "jz_comm_world_free", "jz_knn_build_dist", "jz_knn_rows_dist", "jz_knn_query_dist",
    "jz_knn_dist_stats", "jz_knn_search_host_z", "jz_fof_group_order",
]


class Params(ctypes.Structure):
    _fields_ = [
        ("nmax0", ctypes.c_int32),
        ("coarsen", ctypes.c_int32),
        ("ntarget", ctypes.c_int32),
        ("ngr", ctypes.c_int32),
        ("flags", ctypes.c_uint32),
        ("frame_origin", ctypes.c_float * 3),
        ("frame_extent", ctypes.c_float),
        ("reg_fmax", ctypes.c_int32),
        ("reserved", ctypes.c_int32 * 3),
    ]


class JzError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"jz status {code}: {msg}")
        self.code = code


_lib = None


def lib():
    """Load libjzknn.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                               "(the CUDA extension is required; there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        P, I64, I32, F = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_float
        sig = {
            "jz_knn_build": ([P, I64, P, P, P, P], ctypes.c_int),
            "jz_knn_build_xyzg": ([P, I64, I64, P, P, P, P], ctypes.c_int),
            "jz_knn_build_xq": ([P, I64, P, I64, P, P, P, P], ctypes.c_int),
            "jz_knn_rows": ([P, P], ctypes.c_int),
            "jz_knn_query": ([P, ctypes.c_int, ctypes.c_int, P, P, P, P], ctypes.c_int),
            "jz_knn_free": ([P], None),
            "jz_knn_search_host": ([P, I64, P, P, ctypes.c_int, P, P, P], ctypes.c_int),
            "jz_knn_stage_times": ([P, P, P], ctypes.c_int),
            "jz_set_timing": ([ctypes.c_int], None),
            "jz_last_error": ([], ctypes.c_char_p),
            "jz_morton_keys": ([P, I64, P, P, F, P, P], ctypes.c_int),
            "jz_bucket_by_splitters": ([P, I64, P, I32, P, P, P], ctypes.c_int),
            "jz_pack_by_rank": ([P, I64, I64, P, P, I32, P, P], ctypes.c_int),
            "jz_knn_plane_nodes": ([P, ctypes.c_int, P], ctypes.c_int),
            "jz_knn_query_boxes": ([P, ctypes.c_int, ctypes.c_int, ctypes.c_int, P, P], ctypes.c_int),
            "jz_knn_select_ghosts": ([P, P, I64, ctypes.c_int, I32, P, P, P], ctypes.c_int),
            "jz_knn_pack_ghosts": ([P, P, I32, P, P, P], ctypes.c_int),
            "jz_knn_debug_copy": ([P, ctypes.c_int, ctypes.c_int, P, I64], I64),
            "jz_launch_count": ([], I64),
            "jz_knn_stats": ([P, P], ctypes.c_int),
            "jz_pack_rows": ([P, P, P, I64, I32, P, P, I32, P, P], ctypes.c_int),
            "jz_scatter_rows": ([P, I64, I32, I64, I64, P, P, P], ctypes.c_int),
            "jz_fof": ([P, ctypes.c_float, I32, P, P, P], ctypes.c_int),
            "jz_fof_catalogue": ([P, I64, P, P, P, P, P], ctypes.c_int),
            "jz_comm_unique_id": ([P], ctypes.c_int),
            "jz_comm_init": ([P, ctypes.c_int, ctypes.c_int, P], ctypes.c_int),
            "jz_comm_local_world": ([ctypes.c_int, P], ctypes.c_int),
            "jz_comm_init_local": ([P, ctypes.c_int, P], ctypes.c_int),
            "jz_comm_rank_size": ([P, P, P], ctypes.c_int),
            "jz_comm_free": ([P], None),
            "jz_comm_world_free": ([P], None),
            "jz_knn_build_dist": ([P, P, I64, I64, P, P, P, P], ctypes.c_int),
            "jz_knn_rows_dist": ([P, ctypes.c_int, P], ctypes.c_int),
            "jz_knn_query_dist": ([P, ctypes.c_int, ctypes.c_int, P, P, P, P], ctypes.c_int),
            "jz_knn_dist_stats": ([P, P, P], ctypes.c_int),
            "jz_knn_search_host_z": ([P, I64, P, P, ctypes.c_int, P, P, P, P], ctypes.c_int),
            "jz_fof_group_order": ([P, P, P, P, P], ctypes.c_int),
        }
        for name, (args, res) in sig.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        _lib = L
    return _lib


def check(rc):
    if rc != JZ_OK:
        raise JzError(rc, lib().jz_last_error().decode(errors="replace"))


def stream_ptr(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def box3(box):
    if box is None:
        return None
    if isinstance(box, (int, float)):
        box = (box, box, box)
    return (ctypes.c_float * 3)(*[float(b) for b in box])


def make_params(params=None, **kw):
    p = Params()
    d = dict(params or {})
    d.update(kw)
    for k, v in d.items():
        if k == "frame_origin":
            p.frame_origin = (ctypes.c_float * 3)(*v)
        else:
            setattr(p, k, v)
    return p


def dptr(t: torch.Tensor):
    return ctypes.c_void_p(t.data_ptr())
