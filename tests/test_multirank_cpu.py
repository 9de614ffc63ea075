"""Multi-rank host logic on CPU (gloo, world_size 2): the destination-range
partition (rgnn_partition_dst from librgnn.so), per-rank shards computed by the
fp64 oracle, an all-gather of the owned Y rows and an all-reduce (sum) of dW / dA
must reproduce the unsharded layer exactly as the multi-GPU path composes it
(Y gathered by grouped broadcasts, dW / dA all-reduced, dX
reduce-scattered over the dst ranges)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, model, out_q):
    import sys
    sys.path.insert(0, ROOT)
    import oracle
    import paper_2301_06284_b200 as m
    import synth
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = synth.make_graph(synth.get_config("mutag").scaled(30))
        t = synth.make_tensors(g.V, g.R, 16, 16)
        indeg = np.r_[0, np.cumsum(np.bincount(g.dst, minlength=g.V))]
        bounds = m.partition_dst(indeg, world)
        all_b = [None] * world
        dist.all_gather_object(all_b, [int(x) for x in bounds])
        assert all(b == all_b[0] for b in all_b), "ranks disagree on the partition"
        v0, v1 = int(bounds[rank]), int(bounds[rank + 1])
        G = np.zeros((g.V, 16)); G[v0:v1] = t.dY[v0:v1]
        rows = np.arange(v0, v1)
        if model == "hgt":  # NEXT-3: same partition; dWK, dWQ, dWV, dWa, dWm all-reduced
            h = synth.make_hgt_tensors(g.V, g.R, g.T, 16, 16)
            hw = (h.X, h.WK, h.WQ, h.WV, h.Wa, h.Wm)
            G = np.zeros((g.V, 16)); G[v0:v1] = h.dY[v0:v1]
            Y, _ = oracle.hgt_forward(g.V, g.R, g.src, g.dst, g.etype, g.ntype, *hw, rows=rows)
            grads = oracle.hgt_backward(g.V, g.R, g.src, g.dst, g.etype, g.ntype, *hw, G, v0=v0, v1=v1)
            dW, dA = np.concatenate([x.ravel() for x in grads]), np.zeros(1)
        elif model == "rgat":
            Y, _, _ = oracle.rgat_forward(g.V, g.R, g.src, g.dst, g.etype, t.X, t.W, t.A, rows=rows)
            dW, dA = oracle.rgat_backward(g.V, g.R, g.src, g.dst, g.etype, t.X, t.W, t.A, G, v0=v0, v1=v1)
        else:
            Y = oracle.rgcn_forward(g.V, g.R, g.src, g.dst, g.etype, t.X, t.W, rows=rows)
            dW, _ = oracle.rgcn_backward(g.V, g.R, g.src, g.dst, g.etype, t.X, G, 16, 16, v0=v0, v1=v1)
            dA = np.zeros((g.R, 2, 16))
        # Y_full: every rank's owned rows at its offset (what the grouped broadcasts produce)
        Y_full = torch.zeros(g.V, 16, dtype=torch.float64)
        for k in range(world):
            a, b = int(bounds[k]), int(bounds[k + 1])
            buf = torch.from_numpy(Y.copy()) if k == rank else torch.zeros(b - a, 16, dtype=torch.float64)
            dist.broadcast(buf, src=k)
            Y_full[a:b] = buf
        dWt, dAt = torch.from_numpy(dW), torch.from_numpy(dA)
        dist.all_reduce(dWt)
        dist.all_reduce(dAt)
        if model in ("rgat", "rgcn"):
            # dX (NEXT-2) reduce-scattered over the dst ranges (comm_reduce_rows: one in-place reduce
            # per slice, rooted at the slice's owner): rank k's rows [b_k, b_k+1) become the full dX rows
            if model == "rgat":
                dX = oracle.rgat_dx(g.V, g.R, g.src, g.dst, g.etype, t.X, t.W, t.A, G, v0=v0, v1=v1)
                dXr = oracle.rgat_dx(g.V, g.R, g.src, g.dst, g.etype, t.X, t.W, t.A, t.dY[:, :16])
            else:
                dX = oracle.rgcn_dx(g.V, g.R, g.src, g.dst, g.etype, t.W, G, v0=v0, v1=v1)
                dXr = oracle.rgcn_dx(g.V, g.R, g.src, g.dst, g.etype, t.W, t.dY[:, :16])
            dXt = torch.from_numpy(dX)
            for k in range(world):
                a, b = int(bounds[k]), int(bounds[k + 1])
                sl = dXt[a:b].contiguous()
                dist.reduce(sl, dst=k)
                if k == rank:
                    dXt[a:b] = sl
            np.testing.assert_allclose(dXt[v0:v1].numpy(), dXr[v0:v1], rtol=1e-12, atol=1e-12)
        if rank == 0:
            if model == "hgt":
                Yr, _ = oracle.hgt_forward(g.V, g.R, g.src, g.dst, g.etype, g.ntype, *hw)
                gr = oracle.hgt_backward(g.V, g.R, g.src, g.dst, g.etype, g.ntype, *hw, h.dY)
                dWr, dAr = np.concatenate([x.ravel() for x in gr]), np.zeros(1)
            elif model == "rgat":
                Yr, _, _ = oracle.rgat_forward(g.V, g.R, g.src, g.dst, g.etype, t.X, t.W, t.A)
                dWr, dAr = oracle.rgat_backward(g.V, g.R, g.src, g.dst, g.etype, t.X, t.W, t.A, t.dY[:, :16])
            else:
                Yr = oracle.rgcn_forward(g.V, g.R, g.src, g.dst, g.etype, t.X, t.W)
                dWr, _ = oracle.rgcn_backward(g.V, g.R, g.src, g.dst, g.etype, t.X, t.dY[:, :16], 16, 16)
                dAr = np.zeros_like(dA)
            np.testing.assert_array_equal(Y_full.numpy(), Yr)  # owned rows are computed identically
            np.testing.assert_allclose(dWt.numpy(), dWr, rtol=1e-12, atol=1e-12)
            np.testing.assert_allclose(dAt.numpy(), dAr, rtol=1e-12, atol=1e-12)
            assert bounds[0] == 0 and bounds[-1] == g.V
            out_q.put("ok")
    except Exception as e:  # noqa: BLE001
        out_q.put(f"rank {rank}: {type(e).__name__}: {e}")
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("model", ["rgat", "rgcn", "hgt"])
def test_two_rank_dst_partition_gloo(model):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, model, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    msgs = [q.get(timeout=5) for _ in range(q.qsize())] if not q.empty() else []
    assert all(p.exitcode == 0 for p in procs), msgs
    assert "ok" in msgs, msgs
