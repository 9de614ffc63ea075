"""Shared helpers of the parity tests: run the CUDA path (through the C ABI)
and the fp64 oracle on the same seeded inputs and compare.

Tolerances (reading O19, from north_star's "1e-4 rel / 1e-5 abs"
for fp32 and "2e-2 rel" for bf16):
  |got - ref| <= atol + rtol |ref| elementwise, and ||got-ref||_F <= rtol ||ref||_F
  fp32: rtol 1e-4, atol 1e-5 * max(1, rms(ref))
  bf16: rtol 2e-2, atol 2e-2 * rms(ref)
  per_slice=True (dW [R,K,N], dA [R,2,N]): rms taken over each relation's slice
"""
from __future__ import annotations

import json
import os

import numpy as np

TOL = {"f32": (1e-4, 1e-5, True), "bf16": (2e-2, 2e-2, False)}


def _atol(ref, prec: str, per_slice: bool):
    """per_slice: one rms per leading index -- per relation for dW [R,K,N] / dA [R,2,N], per
    destination row for Y [V,N] (O19: each slice is its own sum with its own scale)."""
    rtol, ascale, floor1 = TOL[prec]
    if per_slice and ref.ndim >= 2:
        rms = np.sqrt(np.mean(ref * ref, axis=tuple(range(1, ref.ndim)), keepdims=True))
    else:
        rms = float(np.sqrt(np.mean(ref * ref)))
    return ascale * (np.maximum(1.0, rms) if floor1 else rms)


def error_ratio(got, ref, prec: str, per_slice: bool = False) -> float:
    """Worst |got - ref| / (atol + rtol |ref|) over the elements (<= 1 passes the elementwise bound)."""
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    if ref.size == 0:
        return 0.0
    bound = _atol(ref, prec, per_slice) + TOL[prec][0] * np.abs(ref)
    err = np.abs(got - ref)
    # exact zeros of the reference (empty rows / relations) must be matched exactly: 0 / 0 -> 0
    return float(np.max(np.where(bound > 0, err / np.where(bound > 0, bound, 1.0), np.where(err > 0, np.inf, 0.0))))


def _log_ratio(got, ref, prec, what, per_slice):
    """RGNN_PARITY_LOG=<file>: append the worst error / bound ratio of this assertion under both
    atol scalings (global rms; per-relation rms) -- the evidence DESIGN.md O19 cites."""
    path = os.environ.get("RGNN_PARITY_LOG")
    if not path:
        return
    rec = {"what": what, "prec": prec, "shape": list(np.shape(ref)),
           "ratio_global": error_ratio(got, ref, prec, False)}
    if np.ndim(ref) >= 2:
        rec["ratio_per_slice"] = error_ratio(got, ref, prec, True)
    r = np.asarray(ref, dtype=np.float64)
    rec["fro"] = float(np.linalg.norm(np.asarray(got, np.float64) - r) / max(np.linalg.norm(r), 1e-300))
    with open(path, "a") as f:
        f.write(json.dumps(rec) + "\n")


def assert_close(got, ref, prec: str, what: str = "", per_slice: bool = False):
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    assert got.shape == ref.shape, (what, got.shape, ref.shape)
    if ref.size == 0:
        return
    _log_ratio(got, ref, prec, what, per_slice)
    rtol = TOL[prec][0]
    atol = _atol(ref, prec, per_slice)
    err = np.abs(got - ref)
    bad = err > atol + rtol * np.abs(ref)
    if bad.any():
        i = np.unravel_index(np.argmax(err - (atol + rtol * np.abs(ref))), ref.shape)
        at = float(np.broadcast_to(atol, ref.shape)[i])
        raise AssertionError(f"{what}: {int(bad.sum())}/{ref.size} elements out of tolerance "
                             f"(prec {prec}, rtol {rtol}, atol {at:.3g}); worst at {i}: got {got[i]!r} ref {ref[i]!r}; "
                             f"max abs err {err.max():.3g}")
    fro = np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-300)
    assert fro <= rtol, f"{what}: relative Frobenius error {fro:.3g} > {rtol}"


def run_gpu(m, g, t, model: str, prec: str, *, slope=0.2, with_w0=False, norm=0, edge_norm=None,
            split_cap=0, dst_range=None, backward=True, materialization="vanilla", want_dx=False):
    """Build the graph and run fwd (+bwd) on the GPU. Returns dict of numpy arrays."""
    import torch
    dev = "cuda"
    v0, v1 = dst_range or (0, g.V)
    G = m.Graph(g.V, g.src, g.dst, g.etype, g.R, norm=norm, edge_norm=edge_norm, row_split_cap=split_cap,
                dst_begin=v0, dst_end=v1, materialization=materialization, build_dx=want_dx)
    Xt = torch.from_numpy(t.X).to(dev)
    X = Xt.to(torch.bfloat16) if prec == "bf16" else Xt
    W = torch.from_numpy(t.W).to(dev)
    A = torch.from_numpy(t.A).to(dev)
    W0 = torch.from_numpy(t.W0).to(dev) if with_w0 else None
    dY = torch.from_numpy(np.ascontiguousarray(t.dY[v0:v1])).to(dev)
    out = {"graph": G}
    K, N = t.W.shape[1], t.W.shape[2]
    ws = m.Workspace(G, model, K, N, prec, dx=want_dx)
    if model == "rgat":
        Y, ws = m.rgat_forward(G, X, W, A, slope, prec=prec, ws=ws)
    else:
        Y, ws = m.rgcn_forward(G, X, W, W0, prec=prec, ws=ws)
    out["Y"] = Y
    if backward:
        res = m.rgnn_backward(G, model, X, W, dY, ws, A=A if model == "rgat" else None, slope=slope, Y=Y,
                              with_w0=with_w0, W0=W0, want_dx=want_dx, prec=prec)
        out.update(dW=res[0], dA=res[1], dW0=res[2])
        if want_dx:
            out["dX"] = res[3]
    torch.cuda.synchronize()
    res = {k: (v.cpu().numpy() if hasattr(v, "cpu") else v) for k, v in out.items() if v is not None}
    res["ws"] = ws
    return res


def bf16_round(a) -> np.ndarray:
    """fp32 -> nearest bf16 (round to nearest even), returned as fp32 values (test input prep)."""
    u = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)


def bf16_inputs(t):
    """The bf16 path's inputs (reading O16): X arrives bf16 and W is rounded to bf16 (RNE); A, dY stay fp32.
    The oracle evaluates the exact layer of these values in fp64, so the LeakyReLU branch (a float decision)
    is taken on the same input values by both sides."""
    import dataclasses
    return dataclasses.replace(t, X=bf16_round(t.X), W=bf16_round(t.W), W0=bf16_round(t.W0))


def run_oracle(oracle, g, t, model: str, *, slope=0.2, with_w0=False, norm=0, edge_norm=None, dst_range=None,
               backward=True, rels=None, prec="f32", want_dx=False):
    if prec == "bf16":
        t = bf16_inputs(t)
    v0, v1 = dst_range or (0, g.V)
    rows = np.arange(v0, v1)
    K, N = t.W.shape[1], t.W.shape[2]
    G = np.zeros((g.V, N)); G[v0:v1] = t.dY[v0:v1]
    out = {}
    if model == "rgat":
        Y, lse, _ = oracle.rgat_forward(g.V, g.R, g.src, g.dst, g.etype, t.X, t.W, t.A, slope=slope, rows=rows)
        out["Y"], out["lse"] = Y, lse
        if backward:
            out["dW"], out["dA"] = oracle.rgat_backward(g.V, g.R, g.src, g.dst, g.etype, t.X, t.W, t.A, G,
                                                        slope=slope, v0=v0, v1=v1, rels=rels)
    else:
        out["Y"] = oracle.rgcn_forward(g.V, g.R, g.src, g.dst, g.etype, t.X, t.W, t.W0 if with_w0 else None,
                                       norm=norm, edge_norm=edge_norm, rows=rows)
        if backward:
            out["dW"], out["dW0"] = oracle.rgcn_backward(g.V, g.R, g.src, g.dst, g.etype, t.X, G, K, N, norm=norm,
                                                         edge_norm=edge_norm, with_w0=with_w0, v0=v0, v1=v1,
                                                         rels=rels)
    if want_dx:
        if model == "rgat":
            out["dX"] = oracle.rgat_dx(g.V, g.R, g.src, g.dst, g.etype, t.X, t.W, t.A, G, slope=slope, v0=v0, v1=v1)
        else:
            out["dX"] = oracle.rgcn_dx(g.V, g.R, g.src, g.dst, g.etype, t.W, G, W0=t.W0 if with_w0 else None,
                                       norm=norm, edge_norm=edge_norm, v0=v0, v1=v1)
    return out
