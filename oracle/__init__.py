"""fp64 CPU oracle for one RGCN / RGAT layer -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this package.  The product path
(paper_2301_06284_b200) never imports it, and it never imports the product.

The arithmetic lives in rgnn_oracle.c (plain C, fp64, per-edge loops; each
function cites the paper passage it follows).  This module only marshals
NumPy arrays through ctypes and builds the shared object with gcc on demand.
Pins: tests/test_oracle_pins.py (DESIGN.md §5 lists which pin covers what).
"""
from __future__ import annotations

import bisect
import ctypes as C
import os
import subprocess
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "rgnn_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

NORM_REL_INDEG, NORM_NONE, NORM_EDGE = 0, 1, 2


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11", "-Wall",
                               "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        i64, i32, f64, vp = C.c_int64, C.c_int32, C.c_double, C.c_void_p
        _lib.oracle_preprocess.restype = i64
        _lib.oracle_preprocess.argtypes = [i64, i64, i32, vp, vp, vp, i64, i64, vp, vp, vp, vp, vp, vp, vp, vp]
        _lib.oracle_rgcn_forward.restype = None
        _lib.oracle_rgcn_forward.argtypes = [i64, i64, i32, i32, i32, vp, vp, vp, vp, vp, vp, i32, vp, i64, vp, vp]
        _lib.oracle_rgat_forward.restype = None
        _lib.oracle_rgat_forward.argtypes = [i64, i64, i32, i32, i32, vp, vp, vp, vp, vp, vp, f64, i32, i64, vp,
                                             vp, vp, vp]
        _lib.oracle_rgat_backward.restype = None
        _lib.oracle_rgat_backward.argtypes = [i64, i64, i32, i32, i32, vp, vp, vp, vp, vp, vp, f64, vp, i64, i64,
                                              vp, vp, vp]
        _lib.oracle_rgcn_backward.restype = None
        _lib.oracle_rgat_dx.argtypes = [i64, i64, i32, i32, i32, vp, vp, vp, vp, vp, vp, f64, vp, i64, i64, vp]
        _lib.oracle_rgat_dx.restype = None
        _lib.oracle_rgcn_dx.argtypes = [i64, i64, i32, i32, i32, vp, vp, vp, vp, vp, i32, vp, vp, i64, i64, vp]
        _lib.oracle_rgcn_dx.restype = None
        _lib.oracle_hgt_forward.argtypes = [i64, i64, i32, i32, i32, i32, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp,
                                            i64, vp, vp, vp]
        _lib.oracle_hgt_forward.restype = None
        _lib.oracle_hgt_backward.argtypes = [i64, i64, i32, i32, i32, i32, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp,
                                             vp, i64, i64, vp, vp, vp, vp, vp]
        _lib.oracle_hgt_backward.restype = None
        _lib.oracle_rgcn_backward.argtypes = [i64, i64, i32, i32, i32, vp, vp, vp, vp, i32, vp, vp, i64, i64, vp,
                                              vp, vp]
        _lib.oracle_num_threads.restype = C.c_int
    return _lib


def _p(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data


def _i32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int32)


def _f64(a) -> Optional[np.ndarray]:
    return None if a is None else np.ascontiguousarray(a, dtype=np.float64)


def num_threads() -> int:
    return int(_load().oracle_num_threads())


class Preprocessed:
    """The oracle's own preprocessing arrays (bit-exact contract, reading O14)."""

    def __init__(self, E_own, perm, src_s, seg, row_ptr, pos, et_slot, cnt):
        self.E_own, self.perm, self.src_s, self.seg = E_own, perm, src_s, seg
        self.row_ptr, self.pos, self.et_slot, self.cnt = row_ptr, pos, et_slot, cnt


class RangeError(ValueError):
    def __init__(self, edge_id: int):
        super().__init__(f"edge {edge_id} has an id out of range")
        self.edge_id = edge_id


def preprocess(V: int, R: int, src, dst, et, v0: int = 0, v1: Optional[int] = None) -> Preprocessed:
    lib = _load()
    src, dst, et = _i32(src), _i32(dst), _i32(et)
    E = src.shape[0]
    v1 = V if v1 is None else v1
    Vown = v1 - v0
    cap = max(E, 1)
    perm = np.empty(cap, np.int32); src_s = np.empty(cap, np.int32); pos = np.empty(cap, np.int32)
    et_slot = np.empty(cap, np.int32); cnt = np.empty(cap, np.int32)
    seg = np.empty(R + 1, np.int32); row_ptr = np.empty(Vown + 1, np.int32)
    bad = np.full(1, -1, np.int64)
    n = lib.oracle_preprocess(V, E, R, _p(src), _p(dst), _p(et), v0, v1, _p(perm), _p(src_s), _p(seg),
                              _p(row_ptr), _p(pos), _p(et_slot), _p(cnt), _p(bad))
    if n < 0:
        raise RangeError(int(bad[0]))
    return Preprocessed(n, perm[:n], src_s[:n], seg, row_ptr, pos[:n], et_slot[:n], cnt[:n])


class Compaction:
    """Compact materialisation tables (Sec. 3.1.3)."""

    def __init__(self, crow_of_pos, csrc, crel, cseg):
        self.crow_of_pos, self.csrc, self.crel, self.cseg = crow_of_pos, csrc, crel, cseg

    @property
    def num_compact(self) -> int:
        return int(self.csrc.shape[0])


def compaction(R: int, pre: Preprocessed) -> Compaction:
    """Compact materialisation: data "merely determined by source
    node features and edge types" is stored "once for each (edge type, unique node
    index) pair", each pair getting "a unique nonnegative integer".
    Reading O15: the integers number the pairs present among the owned edges in
    lexicographic (etype, src) order.  Written out with Python sets and dicts.

    Returns crow_of_pos[p] (compact row of position p), csrc[c] / crel[c] (the
    pair of compact row c) and cseg[r] (compact rows of relation < r)."""
    et_p = np.repeat(np.arange(R, dtype=np.int64), np.diff(pre.seg.astype(np.int64)))  # etype of position p
    keys = list(zip(et_p.tolist(), pre.src_s.tolist()))
    pairs = sorted(set(keys))
    number = {pair: i for i, pair in enumerate(pairs)}
    crow = np.array([number[k] for k in keys], dtype=np.int32)
    csrc = np.array([s for _, s in pairs], dtype=np.int32)
    crel = np.array([r for r, _ in pairs], dtype=np.int32)
    # cseg[r] = number of pairs whose relation is < r; the pairs are sorted, so that count is the
    # bisection point of r in their relation list (same numbers as counting them one by one)
    rel_sorted = [r2 for r2, _ in pairs]
    cseg = np.array([bisect.bisect_left(rel_sorted, r) for r in range(R + 1)], dtype=np.int32)
    return Compaction(crow, csrc, crel, cseg)


def _rows(V: int, rows) -> np.ndarray:
    if rows is None:
        return np.arange(V, dtype=np.int64)
    return np.ascontiguousarray(rows, dtype=np.int64)


def rgcn_forward(V: int, R: int, src, dst, et, X, W, W0=None, norm: int = NORM_REL_INDEG, edge_norm=None,
                 rows: Optional[Sequence[int]] = None) -> np.ndarray:
    """Y[rows] of the RGCN layer, fp64."""
    lib = _load()
    src, dst, et = _i32(src), _i32(dst), _i32(et)
    X, W, W0, en = _f64(X), _f64(W), _f64(W0), _f64(edge_norm)
    R_, K, N = W.shape
    rr = _rows(V, rows)
    Y = np.empty((rr.shape[0], N), np.float64)
    lib.oracle_rgcn_forward(V, src.shape[0], R, K, N, _p(src), _p(dst), _p(et), _p(X), _p(W), _p(W0), norm,
                            _p(en), rr.shape[0], _p(rr), _p(Y))
    return Y


def rgat_forward(V: int, R: int, src, dst, et, X, W, A, slope: float = 0.2, rows=None, stabilize: bool = True,
                 want_alpha: bool = False):
    """(Y[rows], lse[rows], alpha[E] or None) of the RGAT layer, fp64."""
    lib = _load()
    src, dst, et = _i32(src), _i32(dst), _i32(et)
    X, W, A = _f64(X), _f64(W), _f64(A)
    R_, K, N = W.shape
    rr = _rows(V, rows)
    Y = np.empty((rr.shape[0], N), np.float64)
    lse = np.empty(rr.shape[0], np.float64)
    alpha = np.full(src.shape[0], np.nan, np.float64) if want_alpha else None
    lib.oracle_rgat_forward(V, src.shape[0], R, K, N, _p(src), _p(dst), _p(et), _p(X), _p(W), _p(A),
                            float(slope), int(stabilize), rr.shape[0], _p(rr), _p(Y), _p(lse), _p(alpha))
    return Y, lse, alpha


def _mask(R: int, rels) -> Optional[np.ndarray]:
    if rels is None:
        return None
    m = np.zeros(R, np.uint8)
    m[np.asarray(rels, dtype=np.int64)] = 1
    return m


def rgat_backward(V: int, R: int, src, dst, et, X, W, A, G, slope: float = 0.2, v0: int = 0, v1=None, rels=None):
    """(dW [R,K,N], dA [R,2,N]) of L = <Y, G> restricted to dst in [v0, v1)."""
    lib = _load()
    src, dst, et = _i32(src), _i32(dst), _i32(et)
    X, W, A, G = _f64(X), _f64(W), _f64(A), _f64(G)
    R_, K, N = W.shape
    v1 = V if v1 is None else v1
    dW = np.empty((R, K, N), np.float64)
    dA = np.empty((R, 2, N), np.float64)
    m = _mask(R, rels)
    lib.oracle_rgat_backward(V, src.shape[0], R, K, N, _p(src), _p(dst), _p(et), _p(X), _p(W), _p(A),
                             float(slope), _p(G), v0, v1, _p(m), _p(dW), _p(dA))
    return dW, dA


def hgt_forward(V: int, R: int, src, dst, et, ntype, X, WK, WQ, WV, Wa, Wm, rows=None):
    """(Y[rows], lse[rows]) of the HGT layer (NEXT-3, reading O23), fp64."""
    lib = _load()
    src, dst, et, nt = _i32(src), _i32(dst), _i32(et), _i32(ntype)
    X, WK, WQ, WV, Wa, Wm = (_f64(a) for a in (X, WK, WQ, WV, Wa, Wm))
    T, K, N = WK.shape
    rr = _rows(V, rows)
    Y = np.empty((rr.shape[0], N), np.float64)
    lse = np.empty(rr.shape[0], np.float64)
    lib.oracle_hgt_forward(V, src.shape[0], R, T, K, N, _p(src), _p(dst), _p(et), _p(nt), _p(X), _p(WK), _p(WQ),
                           _p(WV), _p(Wa), _p(Wm), rr.shape[0], _p(rr), _p(Y), _p(lse))
    return Y, lse


def hgt_backward(V: int, R: int, src, dst, et, ntype, X, WK, WQ, WV, Wa, Wm, G, v0: int = 0, v1=None):
    """(dWK, dWQ, dWV, dWa, dWm) of the HGT layer's L = <Y, G> restricted to dst in [v0, v1), fp64."""
    lib = _load()
    src, dst, et, nt = _i32(src), _i32(dst), _i32(et), _i32(ntype)
    X, WK, WQ, WV, Wa, Wm, G = (_f64(a) for a in (X, WK, WQ, WV, Wa, Wm, G))
    T, K, N = WK.shape
    v1 = V if v1 is None else v1
    outs = [np.empty((T, K, N)), np.empty((T, K, N)), np.empty((T, K, N)), np.empty((R, N, N)), np.empty((R, N, N))]
    lib.oracle_hgt_backward(V, src.shape[0], R, T, K, N, _p(src), _p(dst), _p(et), _p(nt), _p(X), _p(WK), _p(WQ),
                            _p(WV), _p(Wa), _p(Wm), _p(G), v0, v1, *[_p(o) for o in outs])
    return tuple(outs)


def rgat_dx(V: int, R: int, src, dst, et, X, W, A, G, slope: float = 0.2, v0: int = 0, v1=None) -> np.ndarray:
    """dX [V, K] of L = <Y, G> restricted to dst in [v0, v1) (NEXT-2), fp64."""
    lib = _load()
    src, dst, et = _i32(src), _i32(dst), _i32(et)
    X, W, A, G = _f64(X), _f64(W), _f64(A), _f64(G)
    R_, K, N = W.shape
    v1 = V if v1 is None else v1
    dX = np.empty((V, K), np.float64)
    lib.oracle_rgat_dx(V, src.shape[0], R, K, N, _p(src), _p(dst), _p(et), _p(X), _p(W), _p(A), float(slope),
                       _p(G), v0, v1, _p(dX))
    return dX


def rgcn_dx(V: int, R: int, src, dst, et, W, G, W0=None, norm: int = NORM_REL_INDEG, edge_norm=None, v0: int = 0,
            v1=None) -> np.ndarray:
    """dX [V, K] of the RGCN layer's L = <Y, G> restricted to dst in [v0, v1) (NEXT-2), fp64."""
    lib = _load()
    src, dst, et = _i32(src), _i32(dst), _i32(et)
    W, W0, G, en = _f64(W), _f64(W0), _f64(G), _f64(edge_norm)
    R_, K, N = W.shape
    v1 = V if v1 is None else v1
    dX = np.empty((V, K), np.float64)
    lib.oracle_rgcn_dx(V, src.shape[0], R, K, N, _p(src), _p(dst), _p(et), _p(W), _p(W0), norm, _p(en), _p(G),
                       v0, v1, _p(dX))
    return dX


def rgcn_backward(V: int, R: int, src, dst, et, X, G, K: int, N: int, norm: int = NORM_REL_INDEG, edge_norm=None,
                  with_w0: bool = False, v0: int = 0, v1=None, rels=None):
    """(dW [R,K,N], dW0 [K,N] or None) of L = <Y, G> restricted to dst in [v0, v1)."""
    lib = _load()
    src, dst, et = _i32(src), _i32(dst), _i32(et)
    X, G, en = _f64(X), _f64(G), _f64(edge_norm)
    v1 = V if v1 is None else v1
    dW = np.empty((R, K, N), np.float64)
    dW0 = np.empty((K, N), np.float64) if with_w0 else None
    m = _mask(R, rels)
    lib.oracle_rgcn_backward(V, src.shape[0], R, K, N, _p(src), _p(dst), _p(et), _p(X), norm, _p(en), _p(G),
                             v0, v1, _p(m), _p(dW), _p(dW0))
    return dW, dW0
