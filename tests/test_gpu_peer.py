"""Peer-memory communicator with two real ranks (the comm path had only ever run with
one rank; NCCL cannot put two ranks on one device, CUDA IPC can).

Two processes share the one GPU; each owns a destination range, maps the other's Y_full / signal /
staging buffers with CUDA IPC (rgnn_comm_create_local + rgnn_ipc_export + rgnn_comm_attach_peers,
handles exchanged over gloo), runs the forward -- whose walk stores every finished Y row into both
ranks' Y_full, then a device-side barrier -- and the backward, whose dW / dA are summed through the
staging buffers.  Checks: each rank's Y_full equals the unsharded layer bit for bit (P14), dW / dA
match the unsharded layer and are bit-identical on both ranks, and a second call (epoch 2 of the
barrier, reused buffers) gives the same bits.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, model, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    # one backward kernel on every shard and on the unsharded graph (the default picks per owned graph
    # by its mean (etype, dst) run length; the two kernels agree to the bf16 tolerance, not to 1e-5)
    os.environ["RGNN_BWD_TM"] = "1"
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2301_06284_b200 as m
        import synth
        torch.cuda.set_device(0)
        g = synth.make_graph(synth.get_config("bgs").scaled(4))
        K = N = 64
        t = synth.make_tensors(g.V, g.R, K, N)
        indeg = np.r_[0, np.cumsum(np.bincount(g.dst, minlength=g.V))]
        bounds = m.partition_dst(indeg, world)
        v0, v1 = int(bounds[rank]), int(bounds[rank + 1])
        X = torch.from_numpy(t.X).cuda().to(torch.bfloat16)
        W, A = torch.from_numpy(t.W).cuda(), torch.from_numpy(t.A).cuda()
        dY_full = torch.from_numpy(t.dY).cuda()
        Y_full = torch.full((g.V, N), float("nan"), device="cuda")
        comm = m.PeerComm(bounds, rank, world, Y_full, g.R * K * N + g.R * 2 * N + K * N)
        G = m.Graph(g.V, g.src, g.dst, g.etype, g.R, dst_begin=v0, dst_end=v1, materialization="auto")
        ws = m.Workspace(G, model, K, N, "bf16")
        Y = Y_full[v0:v1]
        dY = dY_full[v0:v1].contiguous()
        outs = []
        for it in range(2):  # the second call runs the barriers' second epoch on reused buffers
            Y_full.fill_(float("nan"))
            if model == "rgat":
                m.rgat_forward(G, X, W, A, 0.2, prec="bf16", ws=ws, Y=Y, comm=comm, Y_full=Y_full)
            else:
                m.rgcn_forward(G, X, W, prec="bf16", ws=ws, Y=Y, comm=comm, Y_full=Y_full)
            dW, dA, _ = m.rgnn_backward(G, model, X, W, dY, ws, A=A if model == "rgat" else None, slope=0.2,
                                        Y=Y, prec="bf16", comm=comm)
            torch.cuda.synchronize()
            outs.append((Y_full.clone(), dW.clone(), dA.clone() if dA is not None else None))
        assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])
        # the unsharded layer in this process
        Gf = m.Graph(g.V, g.src, g.dst, g.etype, g.R, materialization="auto")
        if model == "rgat":
            Yr, wsr = m.rgat_forward(Gf, X, W, A, 0.2, prec="bf16")
        else:
            Yr, wsr = m.rgcn_forward(Gf, X, W, prec="bf16")
        dWr, dAr, _ = m.rgnn_backward(Gf, model, X, W, dY_full, wsr, A=A if model == "rgat" else None, slope=0.2,
                                      Y=Yr, prec="bf16")
        torch.cuda.synchronize()
        Yf, dW, dA = outs[0]
        assert not torch.isnan(Yf).any(), "rows missing from Y_full"
        assert torch.equal(Yf, Yr), "Y_full differs from the unsharded rows"
        rel = float((dW - dWr).norm() / dWr.norm())
        assert rel < 1e-5, f"dW relative difference {rel}"
        if dA is not None:
            rel = float((dA - dAr).norm() / dAr.norm())
            assert rel < 1e-5, f"dA relative difference {rel}"
        sums = [None] * world
        dist.all_gather_object(sums, (dW.double().sum().item(), dW.abs().double().sum().item()))
        assert all(s == sums[0] for s in sums), f"ranks disagree on dW: {sums}"
        q.put("ok")
    except Exception as e:  # noqa: BLE001
        q.put(f"rank {rank}: {type(e).__name__}: {e}")
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("model", ["rgat", "rgcn"])
def test_two_ranks_peer_memory_on_one_gpu(model):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, model, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=280)
    msgs = []
    while not q.empty():
        msgs.append(q.get(timeout=5))
    for p in procs:
        if p.is_alive():
            p.kill()
    assert all(p.exitcode == 0 for p in procs), msgs
    assert msgs.count("ok") == 2, msgs
