"""Compact materialisation (Sec. 3.1.3).

Z and s_src are stored once per unique (etype, src) pair instead of once per
edge.  The tables are bit-exact against oracle.compaction(); the layer is the
same function of its inputs, so outputs match the oracle at the usual tolerance,
and for RGAT -- where each Z row is the same GEMM row either way -- the compact
path reproduces the vanilla path bit for bit.
"""
import numpy as np
import pytest

import oracle
import synth
from parity import assert_close, run_gpu, run_oracle

pytestmark = pytest.mark.gpu


def _graphs():
    return [
        ("toy8", lambda: _toy8()),
        ("rand", lambda: synth.random_graph(300, 5000, 7, seed=1)),
        ("rand-shard", lambda: synth.random_graph(300, 5000, 7, seed=2)),
        ("e0", lambda: synth.random_graph(50, 0, 3, seed=4)),
        ("am/40", lambda: synth.make_graph(synth.get_config("am").scaled(40))),
        ("mag/400", lambda: synth.make_graph(synth.get_config("mag").scaled(400))),
    ]


def _toy8():
    e = np.array([[0, 1, 0], [0, 2, 0], [0, 3, 0], [1, 2, 0], [1, 3, 1], [1, 0, 1], [2, 3, 0], [0, 3, 1]], np.int32)
    return synth.HeteroGraph(4, 2, 1, e[:, 0].copy(), e[:, 1].copy(), e[:, 2].copy(), np.zeros(4, np.int32))


@pytest.mark.parametrize("name,mk", _graphs(), ids=[c[0] for c in _graphs()])
def test_compaction_tables_bit_exact(rgnn, name, mk):
    g = mk()
    v0, v1 = (77, 211) if name == "rand-shard" else (0, g.V)
    G = rgnn.Graph(g.V, g.src, g.dst, g.etype, g.R, dst_begin=v0, dst_end=v1, materialization="compact")
    p = oracle.preprocess(g.V, g.R, g.src, g.dst, g.etype, v0, v1)
    c = oracle.compaction(g.R, p)
    assert G.num_compact == c.num_compact
    a = {k: v.cpu().numpy() for k, v in G.compact_arrays().items()}
    np.testing.assert_array_equal(a["crow_of_pos"], c.crow_of_pos)
    np.testing.assert_array_equal(a["csrc"], c.csrc)
    np.testing.assert_array_equal(a["cseg"], c.cseg)
    # the vanilla tables are unchanged by the option
    np.testing.assert_array_equal(G.arrays()["perm"].cpu().numpy(), p.perm)


CASES = [
    ("rand", lambda: (synth.random_graph(500, 6000, 6, seed=7), 64, 64)),
    ("rand-kn", lambda: (synth.random_graph(400, 3000, 5, seed=8), 128, 64)),
    ("am/40", lambda: (synth.make_graph(synth.get_config("am").scaled(40)), 64, 64)),
    ("mag/400", lambda: (synth.make_graph(synth.get_config("mag").scaled(400)), 128, 128)),
    ("aifb", lambda: (synth.make_graph(synth.get_config("aifb")), 32, 32)),
]


@pytest.mark.parametrize("prec", ["f32", "bf16"])
@pytest.mark.parametrize("model", ["rgat", "rgcn"])
@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_compact_parity(rgnn, case, model, prec):
    g, K, N = case[1]()
    t = synth.make_tensors(g.V, g.R, K, N)
    w0 = model == "rgcn"
    gpu = run_gpu(rgnn, g, t, model, prec, with_w0=w0, materialization="compact")
    assert gpu["graph"].zrows(model) == gpu["graph"].num_compact <= g.E
    ref = run_oracle(oracle, g, t, model, prec=prec, with_w0=w0)
    assert_close(gpu["Y"], ref["Y"], prec, f"compact {model}/{prec} Y")
    assert_close(gpu["dW"], ref["dW"], prec, f"compact {model}/{prec} dW", per_slice=True)
    if model == "rgat":
        assert_close(gpu["dA"], ref["dA"], prec, f"compact {model}/{prec} dA", per_slice=True)
    else:
        assert_close(gpu["dW0"], ref["dW0"], prec, f"compact {model}/{prec} dW0")


@pytest.mark.parametrize("prec", ["f32", "bf16"])
def test_compact_rgat_bit_identical_to_vanilla(rgnn, prec):
    """Same Z rows, same s_src, same walk order: Y, dW and dA are bit identical."""
    g = synth.make_graph(synth.get_config("am").scaled(40))
    t = synth.make_tensors(g.V, g.R, 64, 64)
    a = run_gpu(rgnn, g, t, "rgat", prec)
    b = run_gpu(rgnn, g, t, "rgat", prec, materialization="compact")
    for k in ["Y", "dW", "dA"]:
        np.testing.assert_array_equal(a[k], b[k], err_msg=k)


def test_compact_split_rows_and_shards(rgnn):
    g = synth.make_graph(synth.get_config("wikikg2").scaled(400))
    t = synth.make_tensors(g.V, g.R, 64, 64)
    for model in ["rgat", "rgcn"]:
        gpu = run_gpu(rgnn, g, t, model, "f32", split_cap=8, materialization="compact")
        ref = run_oracle(oracle, g, t, model)
        assert_close(gpu["Y"], ref["Y"], "f32", f"compact split {model} Y")
        assert_close(gpu["dW"], ref["dW"], "f32", f"compact split {model} dW", per_slice=True)
    indeg = np.r_[0, np.cumsum(np.bincount(g.dst, minlength=g.V))]
    b = rgnn.partition_dst(indeg, 2)
    for k in range(2):
        rng = (int(b[k]), int(b[k + 1]))
        gpu = run_gpu(rgnn, g, t, "rgat", "bf16", dst_range=rng, materialization="compact")
        ref = run_oracle(oracle, g, t, "rgat", prec="bf16", dst_range=rng)
        assert_close(gpu["Y"], ref["Y"], "bf16", "compact shard Y")
        assert_close(gpu["dW"], ref["dW"], "bf16", "compact shard dW", per_slice=True)


def test_compact_rejects_bad_option(rgnn):
    g = synth.random_graph(30, 100, 2, seed=1)
    with pytest.raises(rgnn.RgnnError) as ei:
        rgnn.Graph(g.V, g.src, g.dst, g.etype, g.R, materialization=7)
    assert ei.value.status == 1


@pytest.mark.parametrize("name,mk", _graphs()[1:], ids=[c[0] for c in _graphs()[1:]])
def test_auto_materialization_rule(rgnn, name, mk):
    """AUTO (include/rgnn.h): RGCN uses compact rows iff U < E_own, RGAT iff U <= 3/4 E_own;
    COMPACT always, VANILLA never."""
    g = mk()
    c = oracle.compaction(g.R, oracle.preprocess(g.V, g.R, g.src, g.dst, g.etype))
    U = c.num_compact
    Ga = rgnn.Graph(g.V, g.src, g.dst, g.etype, g.R, materialization="auto")
    assert Ga.num_compact == U
    E = Ga.E_own
    assert Ga.zrows("rgcn") == (U if U < E else E)
    assert Ga.zrows("rgat") == (U if 4 * U <= 3 * E else E)
    Gc = rgnn.Graph(g.V, g.src, g.dst, g.etype, g.R, materialization="compact")
    assert Gc.zrows("rgcn") == U and Gc.zrows("rgat") == U
    Gv = rgnn.Graph(g.V, g.src, g.dst, g.etype, g.R)
    assert Gv.zrows("rgcn") == E and Gv.zrows("rgat") == E and Gv.num_compact == 0
