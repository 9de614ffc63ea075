"""Input-feature gradient dX through the C ABI vs the
fp64 oracle (oracle.rgat_dx / rgcn_dx, pinned in test_oracle_pins.py)."""
import numpy as np
import pytest

import oracle
import synth
from parity import assert_close, run_gpu, run_oracle

pytestmark = pytest.mark.gpu

CASES = [
    ("toy", lambda: (synth.HeteroGraph(3, 2, 1, np.array([0, 1, 1, 2], np.int32), np.array([2, 2, 2, 0], np.int32),
                                       np.array([0, 0, 1, 1], np.int32), np.zeros(3, np.int32)), 32, 32)),
    ("rand", lambda: (synth.random_graph(500, 6000, 6, seed=7), 64, 64)),
    ("rand-kn", lambda: (synth.random_graph(400, 3000, 5, seed=8), 128, 64)),
    ("rand-nk", lambda: (synth.random_graph(400, 3000, 5, seed=9), 64, 128)),
    ("mutag/8", lambda: (synth.make_graph(synth.get_config("mutag").scaled(8)), 64, 64)),
    ("aifb", lambda: (synth.make_graph(synth.get_config("aifb")), 32, 32)),
]


@pytest.mark.parametrize("prec", ["f32", "bf16"])
@pytest.mark.parametrize("model", ["rgat", "rgcn"])
@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_dx_parity(rgnn, case, model, prec):
    g, K, N = case[1]()
    t = synth.make_tensors(g.V, g.R, K, N)
    w0 = model == "rgcn"
    gpu = run_gpu(rgnn, g, t, model, prec, with_w0=w0, want_dx=True)
    ref = run_oracle(oracle, g, t, model, prec=prec, with_w0=w0, want_dx=True)
    assert_close(gpu["dX"], ref["dX"], prec, f"{model}/{prec} dX")
    assert_close(gpu["dW"], ref["dW"], prec, f"{model}/{prec} dW", per_slice=True)


@pytest.mark.parametrize("mat", ["compact", "vanilla"])
def test_dx_compact_split_and_shards(rgnn, mat):
    g = synth.make_graph(synth.get_config("am").scaled(40))
    t = synth.make_tensors(g.V, g.R, 64, 64)
    for model in ["rgat", "rgcn"]:
        gpu = run_gpu(rgnn, g, t, model, "bf16", split_cap=8, materialization=mat, want_dx=True)
        ref = run_oracle(oracle, g, t, model, prec="bf16", want_dx=True)
        assert_close(gpu["dX"], ref["dX"], "bf16", f"{mat} {model} dX")
    indeg = np.r_[0, np.cumsum(np.bincount(g.dst, minlength=g.V))]
    b = rgnn.partition_dst(indeg, 3)
    parts = []
    for k in range(3):
        rng = (int(b[k]), int(b[k + 1]))
        gpu = run_gpu(rgnn, g, t, "rgat", "f32", dst_range=rng, materialization=mat, want_dx=True)
        ref = run_oracle(oracle, g, t, "rgat", dst_range=rng, want_dx=True)
        assert_close(gpu["dX"], ref["dX"], "f32", f"shard {k} dX")
        parts.append(gpu["dX"])
    full = run_oracle(oracle, g, t, "rgat", want_dx=True)
    assert_close(sum(parts), full["dX"], "f32", "shard dX sum")


def test_dx_rgcn_without_self_loop_and_norms(rgnn):
    g = synth.random_graph(300, 4000, 5, seed=12)
    t = synth.make_tensors(g.V, g.R, 64, 64)
    en = np.random.default_rng(0).uniform(0.1, 1.0, g.E).astype(np.float32)
    for norm in [0, 1, 2]:
        kw = dict(norm=norm, edge_norm=en if norm == 2 else None)
        gpu = run_gpu(rgnn, g, t, "rgcn", "f32", want_dx=True, **kw)
        ref = run_oracle(oracle, g, t, "rgcn", want_dx=True, **kw)
        assert_close(gpu["dX"], ref["dX"], "f32", f"norm {norm} dX")


def test_dx_deterministic(rgnn):
    g = synth.make_graph(synth.get_config("bgs").scaled(10))
    t = synth.make_tensors(g.V, g.R, 64, 64)
    a = run_gpu(rgnn, g, t, "rgat", "bf16", want_dx=True)
    b = run_gpu(rgnn, g, t, "rgat", "bf16", want_dx=True)
    np.testing.assert_array_equal(a["dX"], b["dX"])


def test_dx_needs_graph_tables(rgnn):
    import torch
    g = synth.random_graph(50, 300, 3, seed=1)
    t = synth.make_tensors(g.V, g.R, 32, 32)
    G = rgnn.Graph(g.V, g.src, g.dst, g.etype, g.R)  # no build_dx
    X = torch.from_numpy(t.X).cuda()
    W = torch.from_numpy(t.W).cuda()
    Y, ws = rgnn.rgcn_forward(G, X, W, prec="f32")
    dY = torch.from_numpy(t.dY).cuda()
    with pytest.raises(rgnn.RgnnError) as ei:
        rgnn.rgnn_backward(G, "rgcn", X, W, dY, ws, Y=Y, want_dx=True, prec="f32")
    assert ei.value.status == 3
