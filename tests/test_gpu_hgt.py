"""HGT forward (reading O23) through the C ABI vs the fp64 oracle
(oracle.hgt_forward, pinned in test_oracle_pins.py)."""
import numpy as np
import pytest

import oracle
import synth
from parity import assert_close, bf16_round

pytestmark = pytest.mark.gpu


def _run(rgnn, g, t, prec, materialization="auto", dst_range=None, split_cap=0):
    import torch
    v0, v1 = dst_range or (0, g.V)
    G = rgnn.Graph(g.V, g.src, g.dst, g.etype, g.R, ntype=g.ntype, num_ntypes=g.T, dst_begin=v0, dst_end=v1,
                   materialization=materialization, row_split_cap=split_cap)
    X = torch.from_numpy(t.X).cuda()
    X = X.to(torch.bfloat16) if prec == "bf16" else X
    Ws = [torch.from_numpy(a).cuda() for a in (t.WK, t.WQ, t.WV, t.Wa, t.Wm)]
    Y, ws = rgnn.hgt_forward(G, X, *Ws, prec=prec)
    torch.cuda.synchronize()
    return Y.cpu().numpy(), ws.saved, G


def _ref(g, t, prec, dst_range=None):
    v0, v1 = dst_range or (0, g.V)
    r = bf16_round if prec == "bf16" else (lambda a: a)
    Y, lse = oracle.hgt_forward(g.V, g.R, g.src, g.dst, g.etype, g.ntype, r(t.X), r(t.WK), r(t.WQ), r(t.WV),
                                r(t.Wa), r(t.Wm), rows=np.arange(v0, v1))
    return Y


CASES = [
    ("rand", lambda: (synth.random_graph(400, 5000, 6, seed=7, T=3), 64, 64)),
    ("rand-kn", lambda: (synth.random_graph(300, 3000, 5, seed=8, T=2), 128, 64)),
    ("rand-nk", lambda: (synth.random_graph(300, 3000, 4, seed=9, T=4), 64, 128)),
    ("mutag/8", lambda: (synth.make_graph(synth.get_config("mutag").scaled(8)), 64, 64)),
    ("aifb", lambda: (synth.make_graph(synth.get_config("aifb")), 32, 32)),
]


@pytest.mark.parametrize("prec", ["f32", "bf16"])
@pytest.mark.parametrize("mat", ["compact", "vanilla"])
@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_hgt_parity(rgnn, case, mat, prec):
    g, K, N = case[1]()
    t = synth.make_hgt_tensors(g.V, g.R, g.T, K, N)
    Y, _, G = _run(rgnn, g, t, prec, materialization=mat)
    assert G.zrows("hgt") == (G.num_compact if mat == "compact" else G.E_own)
    assert_close(Y, _ref(g, t, prec), prec, f"hgt {mat}/{prec} Y")


def test_hgt_split_rows_shards_and_determinism(rgnn):
    g = synth.make_graph(synth.get_config("bgs").scaled(10))
    t = synth.make_hgt_tensors(g.V, g.R, g.T, 64, 64)
    Y, _, _ = _run(rgnn, g, t, "f32", split_cap=8)
    assert_close(Y, _ref(g, t, "f32"), "f32", "hgt split Y")
    Y2, _, _ = _run(rgnn, g, t, "f32", split_cap=8)
    np.testing.assert_array_equal(Y, Y2)
    indeg = np.r_[0, np.cumsum(np.bincount(g.dst, minlength=g.V))]
    b = rgnn.partition_dst(indeg, 2)
    for k in range(2):
        rng = (int(b[k]), int(b[k + 1]))
        Ys, _, _ = _run(rgnn, g, t, "bf16", dst_range=rng)
        assert_close(Ys, _ref(g, t, "bf16", rng), "bf16", f"hgt shard {k}")


def test_hgt_needs_node_types(rgnn):
    import torch
    g = synth.random_graph(40, 200, 3, seed=3, T=2)
    t = synth.make_hgt_tensors(g.V, g.R, g.T, 32, 32)
    G = rgnn.Graph(g.V, g.src, g.dst, g.etype, g.R)
    Ws = [torch.from_numpy(a).cuda() for a in (t.WK, t.WQ, t.WV, t.Wa, t.Wm)]
    with pytest.raises(rgnn.RgnnError) as ei:
        rgnn.hgt_forward(G, torch.from_numpy(t.X).cuda(), *Ws, prec="f32")
    assert ei.value.status == 3


# ---------------------------------------------------------------- backward (NEXT-3)
GRAD_NAMES = ("dWK", "dWQ", "dWV", "dWa", "dWm")


def _run_bwd(rgnn, g, t, prec, materialization="auto", dst_range=None, split_cap=0):
    import torch
    v0, v1 = dst_range or (0, g.V)
    G = rgnn.Graph(g.V, g.src, g.dst, g.etype, g.R, ntype=g.ntype, num_ntypes=g.T, dst_begin=v0, dst_end=v1,
                   materialization=materialization, row_split_cap=split_cap, build_dx=True)
    X = torch.from_numpy(t.X).cuda()
    X = X.to(torch.bfloat16) if prec == "bf16" else X
    Ws = [torch.from_numpy(a).cuda() for a in (t.WK, t.WQ, t.WV, t.Wa, t.Wm)]
    T, K, N = t.WK.shape
    ws = rgnn.Workspace(G, "hgt", K, N, prec, training=True)
    Y, ws = rgnn.hgt_forward(G, X, *Ws, prec=prec, ws=ws)
    dY = torch.from_numpy(t.dY[v0:v1]).cuda().contiguous()
    grads = rgnn.hgt_backward(G, X, *Ws, Y, dY, ws, prec=prec)
    torch.cuda.synchronize()
    return [x.cpu().numpy() for x in grads]


def _ref_bwd(g, t, prec, dst_range=None):
    v0, v1 = dst_range or (0, g.V)
    r = bf16_round if prec == "bf16" else (lambda a: a)
    return oracle.hgt_backward(g.V, g.R, g.src, g.dst, g.etype, g.ntype, r(t.X), r(t.WK), r(t.WQ), r(t.WV),
                               r(t.Wa), r(t.Wm), t.dY, v0=v0, v1=v1)


def _check_grads(got, ref, prec, what):
    for name, a, b in zip(GRAD_NAMES, got, ref):
        assert_close(a, b, prec, f"{what} {name}", per_slice=True)


@pytest.mark.parametrize("prec", ["f32", "bf16"])
@pytest.mark.parametrize("mat", ["compact", "vanilla"])
@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_hgt_backward_parity(rgnn, case, mat, prec):
    g, K, N = case[1]()
    t = synth.make_hgt_tensors(g.V, g.R, g.T, K, N)
    _check_grads(_run_bwd(rgnn, g, t, prec, materialization=mat), _ref_bwd(g, t, prec), prec, f"hgt bwd {mat}/{prec}")


def test_hgt_backward_split_rows_shards_and_determinism(rgnn):
    g = synth.make_graph(synth.get_config("bgs").scaled(10))
    t = synth.make_hgt_tensors(g.V, g.R, g.T, 64, 64)
    got = _run_bwd(rgnn, g, t, "f32", split_cap=8)
    _check_grads(got, _ref_bwd(g, t, "f32"), "f32", "hgt bwd split")
    got2 = _run_bwd(rgnn, g, t, "f32", split_cap=8)
    for a, b in zip(got, got2):
        np.testing.assert_array_equal(a, b)
    # dst-range shards: each shard's gradients match the oracle restricted to its rows, and
    # they sum to the full gradients (what the all-reduce computes across ranks)
    indeg = np.r_[0, np.cumsum(np.bincount(g.dst, minlength=g.V))]
    b = rgnn.partition_dst(indeg, 3)
    full = _ref_bwd(g, t, "bf16")
    acc = None
    for k in range(3):
        rng = (int(b[k]), int(b[k + 1]))
        gs = _run_bwd(rgnn, g, t, "bf16", dst_range=rng)
        _check_grads(gs, _ref_bwd(g, t, "bf16", rng), "bf16", f"hgt bwd shard {k}")
        acc = gs if acc is None else [x + y for x, y in zip(acc, gs)]
    _check_grads(acc, full, "bf16", "hgt bwd shard sum")


def test_hgt_backward_needs_dx_tables(rgnn):
    import torch
    g = synth.random_graph(60, 300, 3, seed=4, T=2)
    t = synth.make_hgt_tensors(g.V, g.R, g.T, 32, 32)
    G = rgnn.Graph(g.V, g.src, g.dst, g.etype, g.R, ntype=g.ntype, num_ntypes=g.T)
    X = torch.from_numpy(t.X).cuda()
    Ws = [torch.from_numpy(a).cuda() for a in (t.WK, t.WQ, t.WV, t.Wa, t.Wm)]
    ws = rgnn.Workspace(G, "hgt", 32, 32, "f32", training=True)
    Y, ws = rgnn.hgt_forward(G, X, *Ws, prec="f32", ws=ws)
    with pytest.raises(rgnn.RgnnError) as ei:
        rgnn.hgt_backward(G, X, *Ws, Y, torch.from_numpy(t.dY).cuda(), ws, prec="f32")
    assert ei.value.status == 3


def _hub_graph():
    """Random graph plus hub runs: 700 edges of relation 1 into node 3 and 130 of relation 0 into
    node 5 (runs longer than one 64-position piece, cut mid-run), and an isolated node type."""
    base = synth.random_graph(200, 1500, 3, seed=11, T=3)
    rng = np.random.Generator(np.random.PCG64(12))
    src = np.r_[base.src, rng.integers(0, 200, 700), rng.integers(0, 200, 130)].astype(np.int32)
    dst = np.r_[base.dst, np.full(700, 3), np.full(130, 5)].astype(np.int32)
    et = np.r_[base.etype, np.full(700, 1), np.zeros(130)].astype(np.int32)
    perm = rng.permutation(src.shape[0])
    return synth.HeteroGraph(V=200, R=3, T=3, src=src[perm], dst=dst[perm], etype=et[perm], ntype=base.ntype,
                             name="hub")


@pytest.mark.parametrize("prec", ["f32", "bf16"])
def test_hgt_backward_long_runs(rgnn, prec):
    g = _hub_graph()
    t = synth.make_hgt_tensors(g.V, g.R, g.T, 64, 64)
    _check_grads(_run_bwd(rgnn, g, t, prec, materialization="vanilla"), _ref_bwd(g, t, prec), prec, "hgt bwd hub")


@pytest.mark.parametrize("prec", ["f32", "bf16"])
def test_hgt_degenerate_graphs(rgnn, prec):
    """E = 0 (Y = 0, all gradients 0), one node with self edges, one edge, a node type without nodes."""
    cases = [synth.random_graph(50, 0, 3, seed=4, T=2), synth.random_graph(1, 20, 2, seed=5, T=1),
             synth.random_graph(30, 1, 2, seed=6, T=3)]
    for g in cases:
        t = synth.make_hgt_tensors(g.V, g.R, g.T, 32, 32)
        Y, _, _ = _run(rgnn, g, t, prec)
        assert_close(Y, _ref(g, t, prec), prec, f"hgt degenerate {g.name} Y")
        _check_grads(_run_bwd(rgnn, g, t, prec), _ref_bwd(g, t, prec), prec, f"hgt degenerate {g.name}")
