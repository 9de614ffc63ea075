"""The library's NCCL path on one GPU (nranks = 1): rgnn_comm_create, the grouped
broadcast gather of Y into Y_full and the in-place all-reduce of dW / dA must
reproduce the communicator-free call bit for bit.  Multi-rank composition is
covered on CPU by tests/test_multirank_cpu.py (gloo)."""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("model", ["rgat", "rgcn"])
def test_single_rank_nccl_matches_no_comm(rgnn, model):
    import torch
    g = synth.make_graph(synth.get_config("bgs").scaled(10))
    t = synth.make_tensors(g.V, g.R, 64, 64)
    G = rgnn.Graph(g.V, g.src, g.dst, g.etype, g.R)
    X = torch.from_numpy(t.X).cuda().to(torch.bfloat16)
    W, A = torch.from_numpy(t.W).cuda(), torch.from_numpy(t.A).cuda()
    dY = torch.from_numpy(t.dY).cuda()
    comm = rgnn.Comm([0, g.V], 0, 1)

    def run(c):
        Y_full = torch.full((g.V, 64), float("nan"), device="cuda") if c else None
        if model == "rgat":
            Y, ws = rgnn.rgat_forward(G, X, W, A, prec="bf16", comm=c, Y_full=Y_full)
        else:
            Y, ws = rgnn.rgcn_forward(G, X, W, prec="bf16", comm=c, Y_full=Y_full)
        dW, dA, _ = rgnn.rgnn_backward(G, model, X, W, dY, ws, A=A if model == "rgat" else None, Y=Y, prec="bf16",
                                       comm=c)
        torch.cuda.synchronize()
        return Y, Y_full, dW, dA

    Y0, _, dW0, dA0 = run(None)
    Y1, Yf, dW1, dA1 = run(comm)
    assert torch.equal(Y0, Y1) and torch.equal(Yf, Y1)
    assert torch.equal(dW0, dW1)
    if model == "rgat":
        assert torch.equal(dA0, dA1)


def test_single_rank_nccl_matches_no_comm_hgt(rgnn):
    import torch
    g = synth.make_graph(synth.get_config("bgs").scaled(10))
    t = synth.make_hgt_tensors(g.V, g.R, g.T, 64, 64)
    G = rgnn.Graph(g.V, g.src, g.dst, g.etype, g.R, ntype=g.ntype, num_ntypes=g.T, build_dx=True)
    X = torch.from_numpy(t.X).cuda().to(torch.bfloat16)
    Ws = [torch.from_numpy(a).cuda() for a in (t.WK, t.WQ, t.WV, t.Wa, t.Wm)]
    dY = torch.from_numpy(t.dY).cuda()
    comm = rgnn.Comm([0, g.V], 0, 1)

    def run(c):
        Y_full = torch.full((g.V, 64), float("nan"), device="cuda") if c else None
        ws = rgnn.Workspace(G, "hgt", 64, 64, "bf16", training=True)
        Y, ws = rgnn.hgt_forward(G, X, *Ws, prec="bf16", ws=ws, comm=c, Y_full=Y_full)
        grads = rgnn.hgt_backward(G, X, *Ws, Y, dY, ws, prec="bf16", comm=c)
        torch.cuda.synchronize()
        return Y, Y_full, grads

    Y0, _, g0 = run(None)
    Y1, Yf, g1 = run(comm)
    assert torch.equal(Y0, Y1) and torch.equal(Yf, Y1)
    for a, b in zip(g0, g1):
        assert torch.equal(a, b)


def test_comm_rejects_mismatched_range(rgnn):
    import torch
    g = synth.random_graph(100, 500, 3, seed=2)
    G = rgnn.Graph(g.V, g.src, g.dst, g.etype, g.R, dst_begin=0, dst_end=50)
    comm = rgnn.Comm([0, g.V], 0, 1)
    X = torch.zeros(g.V, 32, device="cuda")
    W = torch.zeros(g.R, 32, 32, device="cuda")
    with pytest.raises(rgnn.RgnnError) as ei:
        rgnn.rgcn_forward(G, X, W, prec="f32", comm=comm)
    assert ei.value.status == 1


@pytest.mark.parametrize("gather_bf16", [False, True])
def test_single_rank_async_gather_and_join(rgnn, gather_bf16):
    """RGNN_COMM_GATHER_ASYNC (gather on the communicator's own stream, joined before Y_full is
    read) and RGNN_COMM_GATHER_BF16 (bf16 Y_full): Y_full equals Y (rounded to bf16 RNE); the
    backward issued while the gather is pending is unchanged; the whole step captures into a
    CUDA graph (fork on the gather's event, join at the end)."""
    import torch
    g = synth.make_graph(synth.get_config("bgs").scaled(10))
    t = synth.make_tensors(g.V, g.R, 64, 64)
    G = rgnn.Graph(g.V, g.src, g.dst, g.etype, g.R)
    X = torch.from_numpy(t.X).cuda().to(torch.bfloat16)
    W, A = torch.from_numpy(t.W).cuda(), torch.from_numpy(t.A).cuda()
    dY = torch.from_numpy(t.dY).cuda()
    Y0, ws0 = rgnn.rgat_forward(G, X, W, A, prec="bf16")
    dW0, dA0, _ = rgnn.rgnn_backward(G, "rgat", X, W, dY, ws0, A=A, Y=Y0, prec="bf16")
    comm = rgnn.Comm([0, g.V], 0, 1).set_options(gather_async=True, gather_bf16=gather_bf16)
    Y_full = torch.full((g.V, 64), float("nan"), device="cuda", dtype=torch.bfloat16 if gather_bf16 else torch.float32)
    ws = rgnn.Workspace(G, "rgat", 64, 64, "bf16")
    Y = torch.empty(g.V, 64, device="cuda")
    dW = torch.empty_like(dW0)
    dA = torch.empty_like(dA0)

    def step():
        rgnn.rgat_forward(G, X, W, A, prec="bf16", ws=ws, Y=Y, comm=comm, Y_full=Y_full)
        rgnn.rgnn_backward(G, "rgat", X, W, dY, ws, A=A, Y=Y, prec="bf16", comm=comm, dW=dW, dA=dA)
        comm.join()

    step()
    torch.cuda.synchronize()
    assert torch.equal(Y, Y0) and torch.equal(dW, dW0) and torch.equal(dA, dA0)
    assert torch.equal(Y_full, Y0.to(Y_full.dtype))
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        cg = torch.cuda.CUDAGraph()
        with torch.cuda.graph(cg, stream=s):
            step()
    Y_full.fill_(float("nan"))
    cg.replay()
    torch.cuda.synchronize()
    assert torch.equal(Y_full, Y0.to(Y_full.dtype))


def test_single_rank_dx_reduce_scatter(rgnn):
    """dX with a communicator (reduce-scattered over the dst ranges; one rank = identity)."""
    import torch
    g = synth.make_graph(synth.get_config("bgs").scaled(10))
    t = synth.make_tensors(g.V, g.R, 64, 64)
    G = rgnn.Graph(g.V, g.src, g.dst, g.etype, g.R, build_dx=True)
    X = torch.from_numpy(t.X).cuda().to(torch.bfloat16)
    W, A = torch.from_numpy(t.W).cuda(), torch.from_numpy(t.A).cuda()
    dY = torch.from_numpy(t.dY).cuda()
    comm = rgnn.Comm([0, g.V], 0, 1)
    out = []
    for c in (None, comm):
        ws = rgnn.Workspace(G, "rgat", 64, 64, "bf16", dx=True)
        Y, ws = rgnn.rgat_forward(G, X, W, A, prec="bf16", ws=ws)
        out.append(rgnn.rgnn_backward(G, "rgat", X, W, dY, ws, A=A, Y=Y, prec="bf16", want_dx=True, comm=c)[3])
    torch.cuda.synchronize()
    assert torch.equal(out[0], out[1])
