"""Torch-facing wrappers of the C ABI (marshalling only).

PyTorch supplies device memory, streams and process groups; every step of
the layer runs inside librgnn.so (include/rgnn.h).  Names follow the C entry
points: ``rgnn_graph_create`` -> :class:`Graph`, ``rgcn_forward``,
``rgat_forward``, ``rgnn_backward``, ``rgnn_comm_create`` -> :class:`Comm`.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional

import numpy as np
import torch

from . import _binding as B

PREC = {"f32": B.RGNN_F32, "fp32": B.RGNN_F32, "bf16": B.RGNN_BF16}
MODEL = {"rgcn": B.RGNN_RGCN, "rgat": B.RGNN_RGAT, "hgt": B.RGNN_HGT}


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _dev_i32(a, device) -> torch.Tensor:
    if isinstance(a, torch.Tensor):
        return a.to(device=device, dtype=torch.int32).contiguous()
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.int32)).to(device)


def _prec(p) -> int:
    return PREC[p] if isinstance(p, str) else int(p)


def _mat(m) -> int:
    if isinstance(m, str):
        return {"vanilla": B.RGNN_MAT_VANILLA, "compact": B.RGNN_MAT_COMPACT, "auto": B.RGNN_MAT_AUTO}[m]
    return int(m)


def _model(m) -> int:
    return MODEL[m] if isinstance(m, str) else int(m)


class Graph:
    """rgnn_graph_create on caller-owned (torch) device storage."""

    def __init__(self, num_nodes: int, src, dst, etype, num_etypes: int, *, row_ptr=None, ntype=None,
                 num_ntypes: int = 0, norm: int = B.RGNN_NORM_REL_INDEG, edge_norm=None, row_split_cap: int = 0,
                 dst_begin: int = 0, dst_end: Optional[int] = None, materialization="vanilla", build_dx: bool = False,
                 aggregate_first: bool = False, device="cuda", stream=None):
        self.device = torch.device(device)
        self.V, self.R = int(num_nodes), int(num_etypes)
        self.src = _dev_i32(src, self.device)
        self.etype = _dev_i32(etype, self.device)
        self.dst = _dev_i32(dst, self.device) if dst is not None else None
        self.row_ptr_in = _dev_i32(row_ptr, self.device) if row_ptr is not None else None
        self.ntype = _dev_i32(ntype, self.device) if ntype is not None else None
        self.edge_norm = (torch.as_tensor(edge_norm, dtype=torch.float32).to(self.device).contiguous()
                          if edge_norm is not None else None)
        self.dst_begin = int(dst_begin)
        self.dst_end = self.V if dst_end is None else int(dst_end)
        E = int(self.src.shape[0])
        d = B.rgnn_graph_desc(num_nodes=self.V, num_edges=E, num_etypes=self.R, num_ntypes=int(num_ntypes),
                              src=_ptr(self.src), dst=_ptr(self.dst), etype=_ptr(self.etype),
                              row_ptr=_ptr(self.row_ptr_in), ntype=_ptr(self.ntype), edge_norm=_ptr(self.edge_norm),
                              norm=int(norm), row_split_cap=int(row_split_cap), dst_begin=self.dst_begin,
                              dst_end=self.dst_end, materialization=_mat(materialization),
                              flags=(B.RGNN_GRAPH_DX if build_dx else 0) |
                              (B.RGNN_GRAPH_AGGFIRST if aggregate_first else 0))
        self._desc = d
        dev_b, scr_b = C.c_size_t(), C.c_size_t()
        B.call("rgnn_graph_bytes", C.byref(d), C.byref(dev_b), C.byref(scr_b))
        self.storage = torch.empty(max(dev_b.value, 256), dtype=torch.uint8, device=self.device)
        scratch = torch.empty(max(scr_b.value, 256), dtype=torch.uint8, device=self.device)
        h = C.c_void_p()
        self._handle = None
        import time
        t0 = time.perf_counter()
        B.call("rgnn_graph_create", C.byref(d), _ptr(self.storage), dev_b.value, _ptr(scratch), scr_b.value,
               _stream(stream), C.byref(h))  # SYNC
        self.create_ms = 1e3 * (time.perf_counter() - t0)  # the library call alone (buffers preallocated)
        self._handle = h
        del scratch
        v = B.rgnn_graph_view()
        B.call("rgnn_graph_export", h, C.byref(v))
        self.view = v
        self.V_own, self.E_own = int(v.V_own), int(v.E_own)
        self.num_compact = int(v.num_compact)

    @property
    def handle(self):
        return self._handle

    def __del__(self):
        if getattr(self, "_handle", None) is not None:
            B.lib.rgnn_graph_destroy(self._handle)
            self._handle = None

    def _arr(self, ptr, n, dtype) -> torch.Tensor:
        off = int(ptr) - self.storage.data_ptr()
        nbytes = n * torch.tensor([], dtype=dtype).element_size()
        return self.storage[off:off + nbytes].view(dtype)

    def arrays(self) -> dict:
        """Preprocessing outputs as torch views into the graph storage (tests)."""
        v = self.view
        E, Vo, R = int(v.E_own), int(v.V_own), int(v.R)
        i32, f32 = torch.int32, torch.float32
        return {"perm": self._arr(v.perm, E, i32), "src_s": self._arr(v.src_s, E, i32),
                "dst_s": self._arr(v.dst_s, E, i32), "seg": self._arr(v.seg, R + 1, i32),
                "row_ptr": self._arr(v.row_ptr, Vo + 1, i32), "pos": self._arr(v.pos, E, i32),
                "et_slot": self._arr(v.et_slot, E, i32), "inv_c": self._arr(v.inv_c, E, f32),
                "run_ptr": self._arr(v.run_ptr, int(v.num_runs) + 1, i32), "rseg": self._arr(v.rseg, R + 1, i32)}

    def zrows(self, model) -> int:
        """Rows of Z / s_src a layer of `model` materialises (U compact, else E_own)."""
        r = C.c_int64()
        B.call("rgnn_zrows", self._handle, _model(model), C.byref(r))
        return int(r.value)

    def num_pieces(self) -> int:
        """Run pieces (HGT backward / aggregate-first RGCN tables), via the graph view."""
        return int(self.view.num_pieces)

    def piece_arrays(self) -> dict:
        """Aggregate-first tables (graph created with aggregate_first=True), as NumPy arrays (tests)."""
        v = self.view
        E, NP = int(v.E_own), int(v.num_pieces)
        i32, f32 = torch.int32, torch.float32
        return {"piece_ptr": self._arr(v.piece_ptr, NP + 1, i32).cpu().numpy(),
                "slot_piece": self._arr(v.slot_piece, E, i32).cpu().numpy(),
                "slot_w": self._arr(v.slot_w, E, f32).cpu().numpy()}

    def compact_arrays(self) -> dict:
        """Compact materialisation tables (graph created with materialization="compact")."""
        v = self.view
        E, U, R = int(v.E_own), int(v.num_compact), int(v.R)
        i32 = torch.int32
        return {"crow_of_pos": self._arr(v.crow_of_pos, E, i32), "csrc": self._arr(v.csrc, U, i32),
                "cseg": self._arr(v.cseg, R + 1, i32)}


class Comm:
    """rgnn_comm_create: NCCL communicator over the dst-range partition `bounds`."""

    def __init__(self, bounds, rank: int, world: int, group=None):
        import torch.distributed as dist
        idbuf = (C.c_char * 128)()
        if rank == 0:
            B.call("rgnn_comm_unique_id", C.cast(idbuf, C.c_void_p))
        obj = [bytes(idbuf)]
        if world > 1:
            dist.broadcast_object_list(obj, src=0, group=group)
        idbuf = (C.c_char * 128).from_buffer_copy(obj[0])
        b = (C.c_int64 * (world + 1))(*[int(x) for x in bounds])
        h = C.c_void_p()
        B.call("rgnn_comm_create", C.cast(idbuf, C.c_void_p), world, rank, b, C.byref(h))
        self._handle = h
        self.bounds = [int(x) for x in bounds]

    def set_options(self, gather_async: bool = False, gather_bf16: bool = False):
        """rgnn_comm_set_options: asynchronous Y gather (join before reading Y_full) / bf16 Y_full."""
        flags = (B.RGNN_COMM_GATHER_ASYNC if gather_async else 0) | (B.RGNN_COMM_GATHER_BF16 if gather_bf16 else 0)
        B.call("rgnn_comm_set_options", self._handle, flags)
        return self

    def join(self, stream=None):
        """rgnn_comm_join: `stream` waits for the pending asynchronous Y gather."""
        B.call("rgnn_comm_join", self._handle, _stream(stream))

    @property
    def handle(self):
        return self._handle

    def __del__(self):
        if getattr(self, "_handle", None) is not None:
            B.lib.rgnn_comm_destroy(self._handle)
            self._handle = None


class PeerComm(Comm):
    """Peer-memory communicator (rgnn_comm_create_local + rgnn_ipc_export + rgnn_comm_attach_peers):
    every rank's Y_full, signal words and gradient staging buffer are mapped into every process with
    CUDA IPC; the handles are exchanged over the torch.distributed group (any backend, e.g. gloo).
    The forward's walk then stores each finished Y row into every rank's Y_full itself."""

    def __init__(self, bounds, rank: int, world: int, Y_full: torch.Tensor, grad_floats: int, group=None):
        import torch.distributed as dist
        b = (C.c_int64 * (world + 1))(*[int(x) for x in bounds])
        h = C.c_void_p()
        B.call("rgnn_comm_create_local", world, rank, b, C.byref(h))
        self._handle = h
        self.bounds = [int(x) for x in bounds]
        dev = Y_full.device
        self.Y_full = Y_full
        self.sig = torch.zeros(16, dtype=torch.int32, device=dev)       # signal words + epoch
        self.stage = torch.empty(max(int(grad_floats), 1), dtype=torch.float32, device=dev)
        torch.cuda.synchronize(dev)
        mine = []
        for t in (self.Y_full, self.sig, self.stage):
            hb = (C.c_char * 64)()
            off = C.c_int64()
            B.call("rgnn_ipc_export", _ptr(t), C.cast(hb, C.c_void_p), C.byref(off))
            mine.append((bytes(hb), int(off.value)))
        allx = [None] * world
        if world > 1:
            dist.all_gather_object(allx, mine, group=group)
        else:
            allx = [mine]
        handles = (C.c_char * (64 * 3 * world))()
        offs = (C.c_int64 * (3 * world))()
        for k in range(world):
            for j in range(3):
                C.memmove(C.addressof(handles) + (k * 3 + j) * 64, allx[k][j][0], 64)
                offs[k * 3 + j] = allx[k][j][1]
        B.call("rgnn_comm_attach_peers", self._handle, C.cast(handles, C.c_void_p), offs, _ptr(self.Y_full),
               _ptr(self.sig), _ptr(self.stage), self.stage.numel())


def partition_dst(indeg_prefix, nparts: int):
    """rgnn_partition_dst: balanced dst ranges from the in-degree prefix (host)."""
    p = np.ascontiguousarray(indeg_prefix, dtype=np.int64)
    V = p.shape[0] - 1
    out = np.zeros(nparts + 1, np.int64)
    B.call("rgnn_partition_dst", V, p.ctypes.data_as(C.POINTER(C.c_int64)), nparts,
           out.ctypes.data_as(C.POINTER(C.c_int64)))
    return out


class Workspace:
    """Workspace + saved buffers sized by rgnn_workspace_bytes (reused across calls)."""

    def __init__(self, g: Graph, model, d_in: int, d_out: int, prec, training: bool = True, dx: bool = False):
        ws, sv = C.c_size_t(), C.c_size_t()
        mode = B.RGNN_WS_DX if dx else int(training)
        B.call("rgnn_workspace_bytes", g.handle, _model(model), d_in, d_out, _prec(prec), mode,
               C.byref(ws), C.byref(sv))
        self.dx = dx
        self.ws = torch.empty(max(ws.value, 256), dtype=torch.uint8, device=g.device)
        self.saved = torch.empty(max(sv.value, 256), dtype=torch.uint8, device=g.device)
        self.key = (_model(model), d_in, d_out, _prec(prec))


def _check_x(X: torch.Tensor, prec: int):
    want = torch.bfloat16 if prec == B.RGNN_BF16 else torch.float32
    if X.dtype != want or not X.is_contiguous() or not X.is_cuda:
        raise ValueError(f"X must be a contiguous CUDA {want} tensor")


def rgcn_forward(g: Graph, X: torch.Tensor, W: torch.Tensor, W0: Optional[torch.Tensor] = None, *, prec="f32",
                 ws: Optional[Workspace] = None, Y: Optional[torch.Tensor] = None, comm: Optional[Comm] = None,
                 Y_full: Optional[torch.Tensor] = None, stream=None):
    p = _prec(prec)
    _check_x(X, p)
    R, K, N = W.shape
    ws = ws or Workspace(g, "rgcn", K, N, p)
    Y = Y if Y is not None else torch.empty(g.V_own, N, dtype=torch.float32, device=g.device)
    B.call("rgcn_forward", g.handle, K, N, p, _ptr(X), _ptr(W), _ptr(W0), _ptr(Y), _ptr(ws.saved), _ptr(ws.ws),
           ws.ws.numel(), comm.handle if comm else None, _ptr(Y_full), _stream(stream))
    return Y, ws


def rgat_forward(g: Graph, X: torch.Tensor, W: torch.Tensor, A: torch.Tensor, slope: float = 0.2, *, prec="bf16",
                 ws: Optional[Workspace] = None, Y: Optional[torch.Tensor] = None, comm: Optional[Comm] = None,
                 Y_full: Optional[torch.Tensor] = None, stream=None):
    p = _prec(prec)
    _check_x(X, p)
    R, K, N = W.shape
    ws = ws or Workspace(g, "rgat", K, N, p)
    Y = Y if Y is not None else torch.empty(g.V_own, N, dtype=torch.float32, device=g.device)
    B.call("rgat_forward", g.handle, K, N, p, _ptr(X), _ptr(W), _ptr(A), float(slope), _ptr(Y), _ptr(ws.saved),
           _ptr(ws.ws), ws.ws.numel(), comm.handle if comm else None, _ptr(Y_full), _stream(stream))
    return Y, ws


def hgt_forward(g: Graph, X: torch.Tensor, WK: torch.Tensor, WQ: torch.Tensor, WV: torch.Tensor, Wa: torch.Tensor,
                Wm: torch.Tensor, *, prec="bf16", ws: Optional[Workspace] = None, Y: Optional[torch.Tensor] = None,
                comm: Optional[Comm] = None, Y_full: Optional[torch.Tensor] = None, stream=None):
    """hgt_forward (NEXT-3): WK/WQ/WV [T, d_in, d_out], Wa/Wm [R, d_out, d_out]."""
    p = _prec(prec)
    _check_x(X, p)
    T, K, N = WK.shape
    ws = ws or Workspace(g, "hgt", K, N, p)
    Y = Y if Y is not None else torch.empty(g.V_own, N, dtype=torch.float32, device=g.device)
    B.call("hgt_forward", g.handle, K, N, p, _ptr(X), _ptr(WK), _ptr(WQ), _ptr(WV), _ptr(Wa), _ptr(Wm), _ptr(Y),
           _ptr(ws.saved), _ptr(ws.ws), ws.ws.numel(), comm.handle if comm else None, _ptr(Y_full), _stream(stream))
    return Y, ws


def hgt_backward(g: Graph, X: torch.Tensor, WK: torch.Tensor, WQ: torch.Tensor, WV: torch.Tensor, Wa: torch.Tensor,
                 Wm: torch.Tensor, Y: torch.Tensor, dY: torch.Tensor, ws: Workspace, *, prec="bf16",
                 comm: Optional[Comm] = None, stream=None):
    """hgt_backward (NEXT-3): returns (dWK, dWQ, dWV, dWa, dWm).  ws must come from the forward
    (Workspace(..., training=True)); the graph must be built with build_dx=True and node types."""
    p = _prec(prec)
    _check_x(X, p)
    T, K, N = WK.shape
    R = Wa.shape[0]
    dev = g.device
    outs = [torch.empty(T, K, N, dtype=torch.float32, device=dev) for _ in range(3)] + \
           [torch.empty(R, N, N, dtype=torch.float32, device=dev) for _ in range(2)]
    B.call("hgt_backward", g.handle, K, N, p, _ptr(X), _ptr(WK), _ptr(WQ), _ptr(WV), _ptr(Wa), _ptr(Wm), _ptr(Y),
           _ptr(dY), _ptr(ws.saved), *[_ptr(o) for o in outs], _ptr(ws.ws), ws.ws.numel(),
           comm.handle if comm else None, _stream(stream))
    return tuple(outs)


def rgnn_backward(g: Graph, model, X: torch.Tensor, W: torch.Tensor, dY: torch.Tensor, ws: Workspace, *,
                  A: Optional[torch.Tensor] = None, slope: float = 0.2, Y: Optional[torch.Tensor] = None,
                  with_w0: bool = False, W0: Optional[torch.Tensor] = None, want_dx: bool = False, prec="bf16",
                  comm: Optional[Comm] = None, dW=None, dA=None, dW0=None, dX=None, stream=None):
    """rgnn_backward.  Returns (dW, dA, dW0) or, with want_dx, (dW, dA, dW0, dX [V, d_in])."""
    p, m = _prec(prec), _model(model)
    R, K, N = W.shape
    dW = dW if dW is not None else torch.empty(R, K, N, dtype=torch.float32, device=g.device)
    if m == B.RGNN_RGAT and dA is None:
        dA = torch.empty(R, 2, N, dtype=torch.float32, device=g.device)
    if with_w0 and dW0 is None:
        dW0 = torch.empty(K, N, dtype=torch.float32, device=g.device)
    if want_dx and dX is None:
        dX = torch.empty(g.V, K, dtype=torch.float32, device=g.device)
    B.call("rgnn_backward", g.handle, m, K, N, p, _ptr(X), _ptr(W), _ptr(W0), _ptr(A), float(slope), _ptr(Y),
           _ptr(dY), _ptr(ws.saved), _ptr(dW), _ptr(dA), _ptr(dW0) if with_w0 else None,
           _ptr(dX) if want_dx else None, _ptr(ws.ws), ws.ws.numel(), comm.handle if comm else None, _stream(stream))
    return (dW, dA, dW0, dX) if want_dx else (dW, dA, dW0)
