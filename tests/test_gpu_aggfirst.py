"""Aggregate-first RGCN forward.

RGCN is linear in its messages: Y_v = sum_r (1/c_{v,r}) (sum_{e in run(r,v)} x_src) W_r,
so the library can sum x_src over each (etype, dst) run first (runs cut into pieces of <= 64
positions) and run the typed GEMM over the pieces instead of the edges (graph flag
RGNN_GRAPH_AGGFIRST).  The piece tables are integer data, checked bit-exactly against a NumPy
construction from the oracle's preprocessing; Y is the same layer, checked against the fp64
oracle at the usual tolerance; the backward is unchanged by the option.
"""
import numpy as np
import pytest

import oracle
import synth
from parity import assert_close, run_oracle

pytestmark = pytest.mark.gpu

PIECE = 64  # kPieceRows


def _pieces(g, v0=0, v1=None):
    """Pieces from the oracle's preprocessing: each (etype, dst) run cut every 64 positions from its start."""
    p = oracle.preprocess(g.V, g.R, g.src, g.dst, g.etype, v0, v1)
    keys = g.etype[p.perm].astype(np.int64) * g.V + g.dst[p.perm]
    E = p.E_own
    heads = np.r_[True, keys[1:] != keys[:-1]] if E else np.zeros(0, bool)
    run_start = np.maximum.accumulate(np.where(heads, np.arange(E), 0)) if E else np.zeros(0, np.int64)
    cut = heads | ((np.arange(E) - run_start) % PIECE == 0)  # every 64 positions from the run start
    starts = np.flatnonzero(cut)
    piece_of_pos = np.cumsum(cut) - 1
    return p, starts, piece_of_pos


CASES = [
    ("rand", lambda: synth.random_graph(500, 6000, 6, seed=7)),
    ("am/40", lambda: synth.make_graph(synth.get_config("am").scaled(40))),
    ("wikikg2/100", lambda: synth.make_graph(synth.get_config("wikikg2").scaled(100))),
    ("mag/400", lambda: synth.make_graph(synth.get_config("mag").scaled(400))),
    ("hub", lambda: synth.HeteroGraph(300, 2, 1, np.arange(1000, dtype=np.int32) % 300,
                                      np.zeros(1000, np.int32), (np.arange(1000) % 2).astype(np.int32),
                                      np.zeros(300, np.int32))),
]


@pytest.mark.parametrize("name,mk", CASES, ids=[c[0] for c in CASES])
def test_piece_tables_bit_exact(rgnn, name, mk):
    g = mk()
    G = rgnn.Graph(g.V, g.src, g.dst, g.etype, g.R, aggregate_first=True)
    p, starts, piece_of_pos = _pieces(g)
    assert G.num_pieces() == starts.shape[0]
    t = G.piece_arrays()
    np.testing.assert_array_equal(t["piece_ptr"], np.r_[starts, p.E_own].astype(np.int32))
    slot_piece = piece_of_pos[p.pos]
    np.testing.assert_array_equal(t["slot_piece"], slot_piece)
    dst_slot = g.dst[p.perm][p.pos]
    first = np.r_[True, (slot_piece[1:] != slot_piece[:-1]) | (dst_slot[1:] != dst_slot[:-1])]
    np.testing.assert_array_equal(t["slot_w"], first.astype(np.float32))


@pytest.mark.parametrize("prec", ["f32", "bf16"])
@pytest.mark.parametrize("case", [("rand", 64, 64), ("am/40", 64, 64), ("wikikg2/100", 64, 64), ("mag/400", 128, 128),
                                  ("hub", 32, 32)], ids=lambda c: c[0] if isinstance(c, tuple) else c)
def test_aggregate_first_parity(rgnn, case, prec):
    import torch
    name, K, N = case
    g = dict(CASES)[name]()
    t = synth.make_tensors(g.V, g.R, K, N)
    for w0, norm in ((False, 0), (True, 0), (False, 2)):
        en = np.random.default_rng(0).uniform(0.1, 1.0, g.E).astype(np.float32) if norm == 2 else None
        G = rgnn.Graph(g.V, g.src, g.dst, g.etype, g.R, aggregate_first=True, row_split_cap=16, norm=norm,
                       edge_norm=en)
        X = torch.from_numpy(t.X).cuda()
        X = X.to(torch.bfloat16) if prec == "bf16" else X
        W = torch.from_numpy(t.W).cuda()
        W0 = torch.from_numpy(t.W0).cuda() if w0 else None
        Y, ws = rgnn.rgcn_forward(G, X, W, W0, prec=prec)
        dW, _, dW0 = rgnn.rgnn_backward(G, "rgcn", X, W, torch.from_numpy(t.dY).cuda(), ws, with_w0=w0, W0=W0,
                                        prec=prec)
        ref = run_oracle(oracle, g, t, "rgcn", prec=prec, with_w0=w0, norm=norm, edge_norm=en)
        assert_close(Y.cpu().numpy(), ref["Y"], prec, f"aggregate-first {name} Y (W0 {w0}, norm {norm})")
        assert_close(dW.cpu().numpy(), ref["dW"], prec, f"aggregate-first {name} dW", per_slice=True)


def test_aggregate_first_shards_match(rgnn):
    """Sharded aggregate-first rows equal the unsharded ones bit for bit (pieces depend only on the run)."""
    import torch
    g = synth.make_graph(synth.get_config("wikikg2").scaled(200))
    t = synth.make_tensors(g.V, g.R, 64, 64)
    X = torch.from_numpy(t.X).cuda().to(torch.bfloat16)
    W = torch.from_numpy(t.W).cuda()
    Yf, _ = rgnn.rgcn_forward(rgnn.Graph(g.V, g.src, g.dst, g.etype, g.R, aggregate_first=True), X, W, prec="bf16")
    indeg = np.r_[0, np.cumsum(np.bincount(g.dst, minlength=g.V))]
    b = rgnn.partition_dst(indeg, 3)
    ys = []
    for k in range(3):
        G = rgnn.Graph(g.V, g.src, g.dst, g.etype, g.R, aggregate_first=True, dst_begin=int(b[k]), dst_end=int(b[k + 1]))
        ys.append(rgnn.rgcn_forward(G, X, W, prec="bf16")[0])
    assert torch.equal(torch.cat(ys), Yf)
