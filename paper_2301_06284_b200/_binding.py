"""ctypes binding of librgnn.so -- argument marshalling only.

Function names mirror include/rgnn.h one to one.  Every step of the layer
runs in the library's CUDA kernels; this module has no fallback: if the
shared library is missing it raises ImportError.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "librgnn.so")

RGNN_OK, RGNN_E_INVALID_ARG, RGNN_E_RANGE, RGNN_E_UNSUPPORTED, RGNN_E_WORKSPACE, RGNN_E_CUDA, RGNN_E_NCCL = range(7)
RGNN_F32, RGNN_BF16 = 0, 1
RGNN_NORM_REL_INDEG, RGNN_NORM_NONE, RGNN_NORM_EDGE = 0, 1, 2
RGNN_RGCN, RGNN_RGAT, RGNN_HGT = 0, 1, 2
RGNN_MAT_VANILLA, RGNN_MAT_COMPACT, RGNN_MAT_AUTO = 0, 1, 2
RGNN_GRAPH_DX = 1
RGNN_GRAPH_AGGFIRST = 2
RGNN_WS_DX = 3
RGNN_COMM_GATHER_ASYNC = 1
RGNN_COMM_GATHER_BF16 = 2

STATUS_NAMES = {0: "RGNN_OK", 1: "RGNN_E_INVALID_ARG", 2: "RGNN_E_RANGE", 3: "RGNN_E_UNSUPPORTED",
                4: "RGNN_E_WORKSPACE", 5: "RGNN_E_CUDA", 6: "RGNN_E_NCCL"}


class rgnn_graph_desc(C.Structure):
    _fields_ = [("num_nodes", C.c_int64), ("num_edges", C.c_int64), ("num_etypes", C.c_int32),
                ("num_ntypes", C.c_int32), ("src", C.c_void_p), ("dst", C.c_void_p), ("etype", C.c_void_p),
                ("row_ptr", C.c_void_p), ("ntype", C.c_void_p), ("edge_norm", C.c_void_p), ("norm", C.c_int32),
                ("row_split_cap", C.c_int32), ("dst_begin", C.c_int64), ("dst_end", C.c_int64),
                ("materialization", C.c_int32), ("flags", C.c_int32)]


class rgnn_graph_view(C.Structure):
    _fields_ = [("V", C.c_int64), ("V_own", C.c_int64), ("dst_begin", C.c_int64), ("E_own", C.c_int64),
                ("num_runs", C.c_int64), ("num_tiles", C.c_int64), ("num_items", C.c_int64),
                ("num_split_rows", C.c_int64), ("R", C.c_int32),
                ("perm", C.c_void_p), ("src_s", C.c_void_p), ("dst_s", C.c_void_p), ("seg", C.c_void_p),
                ("row_ptr", C.c_void_p), ("pos", C.c_void_p), ("et_slot", C.c_void_p), ("inv_c", C.c_void_p),
                ("run_ptr", C.c_void_p), ("rseg", C.c_void_p), ("seg_host", C.POINTER(C.c_int32)),
                ("num_compact", C.c_int64), ("crow_of_pos", C.c_void_p), ("csrc", C.c_void_p), ("cseg", C.c_void_p),
                ("num_pieces", C.c_int64), ("piece_ptr", C.c_void_p),
                ("slot_piece", C.c_void_p), ("slot_w", C.c_void_p)]


class RgnnError(RuntimeError):
    def __init__(self, status: int, fn: str, msg: str):
        super().__init__(f"{fn} -> {STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: run `make` (or __graft_entry__.build()) -- there is no fallback")

lib = C.CDLL(LIB_PATH)

_vp, _i32, _i64, _f32, _sz = C.c_void_p, C.c_int32, C.c_int64, C.c_float, C.c_size_t
_SIGS = {
    "rgnn_graph_bytes": [C.POINTER(rgnn_graph_desc), C.POINTER(_sz), C.POINTER(_sz)],
    "rgnn_graph_create": [C.POINTER(rgnn_graph_desc), _vp, _sz, _vp, _sz, _vp, C.POINTER(_vp)],
    "rgnn_graph_export": [_vp, C.POINTER(rgnn_graph_view)],
    "rgnn_workspace_bytes": [_vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(_sz), C.POINTER(_sz)],
    "rgcn_forward": [_vp, C.c_int, C.c_int, C.c_int, _vp, _vp, _vp, _vp, _vp, _vp, _sz, _vp, _vp, _vp],
    "rgat_forward": [_vp, C.c_int, C.c_int, C.c_int, _vp, _vp, _vp, _f32, _vp, _vp, _vp, _sz, _vp, _vp, _vp],
    "rgnn_backward": [_vp, C.c_int, C.c_int, C.c_int, C.c_int, _vp, _vp, _vp, _vp, _f32, _vp, _vp, _vp, _vp, _vp,
                      _vp, _vp, _vp, _sz, _vp, _vp],
    "rgnn_comm_unique_id": [_vp],
    "rgnn_comm_create": [_vp, C.c_int, C.c_int, C.POINTER(_i64), C.POINTER(_vp)],
    "rgnn_comm_set_options": [_vp, C.c_int],
    "rgnn_comm_create_local": [C.c_int, C.c_int, C.POINTER(_i64), C.POINTER(_vp)],
    "rgnn_ipc_export": [_vp, _vp, C.POINTER(_i64)],
    "rgnn_comm_attach_peers": [_vp, _vp, C.POINTER(_i64), _vp, _vp, _vp, _sz],
    "rgnn_comm_join": [_vp, _vp],
    "rgnn_partition_dst": [_i64, C.POINTER(_i64), C.c_int, C.POINTER(_i64)],
    "rgnn_zrows": [_vp, C.c_int, C.POINTER(_i64)],
    "hgt_forward": [_vp, C.c_int, C.c_int, C.c_int, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _sz, _vp, _vp, _vp],
    "hgt_backward": [_vp, C.c_int, C.c_int, C.c_int] + [_vp] * 14 + [_vp, _sz, _vp, _vp],
}
for _name, _args in _SIGS.items():
    _f = getattr(lib, _name)
    _f.argtypes = _args
    _f.restype = C.c_int
lib.rgnn_graph_destroy.argtypes = [_vp]
lib.rgnn_graph_destroy.restype = None
lib.rgnn_comm_destroy.argtypes = [_vp]
lib.rgnn_comm_destroy.restype = None
lib.rgnn_launch_count.argtypes = []
lib.rgnn_launch_count.restype = C.c_uint64
lib.rgnn_last_error.argtypes = []
lib.rgnn_last_error.restype = C.c_char_p
lib.rgnn_version.argtypes = []
lib.rgnn_version.restype = C.c_char_p
lib.rgnn_profile_enable.argtypes = [C.c_int]
lib.rgnn_profile_enable.restype = None
lib.rgnn_profile_read.argtypes = [C.c_char_p, C.POINTER(C.c_double), C.POINTER(C.c_int64), C.c_int]
lib.rgnn_profile_read.restype = C.c_int

EXPORTED = sorted(list(_SIGS) + ["rgnn_graph_destroy", "rgnn_comm_destroy", "rgnn_launch_count", "rgnn_last_error",
                                 "rgnn_version", "rgnn_profile_enable", "rgnn_profile_read"])


def check(status: int, fn: str) -> None:
    if status != RGNN_OK:
        raise RgnnError(status, fn, lib.rgnn_last_error().decode(errors="replace"))


def call(name: str, *args) -> None:
    check(getattr(lib, name)(*args), name)


def launch_count() -> int:
    return int(lib.rgnn_launch_count())


def version() -> str:
    return lib.rgnn_version().decode()


def profile_enable(on: bool = True) -> None:
    lib.rgnn_profile_enable(1 if on else 0)


def profile_read(max_phases: int = 32) -> dict:
    """{phase: (total_ms, launches)} since the last read (SYNC)."""
    names = C.create_string_buffer(32 * max_phases)
    ms = (C.c_double * max_phases)()
    cnt = (C.c_int64 * max_phases)()
    n = lib.rgnn_profile_read(names, ms, cnt, max_phases)
    raw = names.raw
    return {raw[32 * i:32 * i + 32].split(b"\0", 1)[0].decode(): (ms[i], int(cnt[i])) for i in range(n)}
