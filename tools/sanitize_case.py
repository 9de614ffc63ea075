"""One tiny invocation of every hot-path kernel family, for compute-sanitizer
(tests/test_gpu_sanitize.py runs it under memcheck / racecheck / synccheck / initcheck).

Covers: preprocessing (radix sort, tables, compact rows, dX / HGT tables), the tcgen05 typed
GEMM (k_gemm_fwd_tc), the narrow and wide forward walks (k_aggregate_narrow, k_aggregate,
k_aggregate_ring, k_merge), the fused tcgen05 backward (k_bwd_fused_tc), the unfused backward
with the tcgen05 dW GEMM (k_gemm_dw_tc), the tf32 GEMM and source walks of dX
(k_gemm_fwd_tf32, k_dx_walk) and the HGT walks.  Arguments: "fused" (default), "unfused" or "f32"
(the fp32 layer: 3xTF32 typed GEMM k_gemm_fwd_tf32x3 and dW GEMM k_gemm_dw_tf32x3, fp32 walks), then
"full" (default) or "rgat64" (the RGAT d = 64 forward + backward + dX only: racecheck's scope).
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2301_06284_b200 as m  # noqa: E402
import synth  # noqa: E402


def main(scope="full", prec="bf16"):
    torch.cuda.set_device(0)
    n0 = m.launch_count()
    # full MUTAG shape: the fused backward's chunks (>= 2 per SM) then span more stages than its ring
    # holds, so every stage slot is refilled (the WAR / WAW paths racecheck must see)
    g = synth.make_graph(synth.get_config("mutag"))
    for d in ((64,) if scope == "rgat64" else (64, 128)):
        t = synth.make_tensors(g.V, g.R, d, d)
        G = m.Graph(g.V, g.src, g.dst, g.etype, g.R, ntype=g.ntype, num_ntypes=g.T, materialization="auto",
                    build_dx=True, row_split_cap=16)
        X = torch.from_numpy(t.X).cuda()
        X = X.to(torch.bfloat16) if prec == "bf16" else X
        W = torch.from_numpy(t.W).cuda()
        A = torch.from_numpy(t.A).cuda()
        dY = torch.from_numpy(t.dY).cuda()
        ws = m.Workspace(G, "rgat", d, d, prec, dx=True)
        Y, ws = m.rgat_forward(G, X, W, A, 0.2, prec=prec, ws=ws)
        m.rgnn_backward(G, "rgat", X, W, dY, ws, A=A, slope=0.2, Y=Y, prec=prec, want_dx=True)
        if scope == "rgat64":  # racecheck: the mbarrier pipelines of the RGAT path only (minutes per kernel)
            continue
        wr = m.Workspace(G, "rgcn", d, d, prec)
        Yr, wr = m.rgcn_forward(G, X, W, prec=prec, ws=wr)
        m.rgnn_backward(G, "rgcn", X, W, dY, wr, prec=prec)
        if d == 64 and prec == "bf16":
            h = synth.make_hgt_tensors(g.V, g.R, g.T, d, d)
            Hw = [torch.from_numpy(a).cuda() for a in (h.WK, h.WQ, h.WV, h.Wa, h.Wm)]
            wh = m.Workspace(G, "hgt", d, d, "bf16", training=True)
            Yh, wh = m.hgt_forward(G, X, *Hw, prec="bf16", ws=wh)
            m.hgt_backward(G, X, *Hw, Yh, torch.from_numpy(h.dY).cuda(), wh, prec="bf16")
    torch.cuda.synchronize()
    print("sanitize case ok", np.float64(Y.float().abs().sum().item()), f"{m.launch_count() - n0} kernel launches")


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "unfused":
        os.environ["RGNN_DISABLE_FUSED_BWD"] = "1"
    main(sys.argv[2] if len(sys.argv) > 2 else "full", "f32" if len(sys.argv) > 1 and sys.argv[1] == "f32" else "bf16")
