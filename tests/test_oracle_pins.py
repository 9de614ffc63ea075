"""Pins for the fp64 oracle (run with -m "not gpu").

Each test pins the oracle to something other than itself:
hand-derived worked example, brute force with a different algorithm, dense
NumPy / SciPy / torch library routines, closed forms, special cases, finite
differences and invariances.  A plausible slip in the oracle (dropped term,
wrong sign/index, transposed W, wrong concat order, per-relation instead of
per-destination softmax, c over the wrong set) fails at least one of these.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle
import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden", "toy_graph.json")


def toy():
    with open(GOLD) as f:
        g = json.load(f)
    e = np.array(g["edges_src_dst_etype"], np.int32)
    return g, e[:, 0], e[:, 1], e[:, 2], np.array(g["X"], float), np.array(g["W"], float), np.array(g["A"], float)


# ---------------------------------------------------------------- golden toy
def test_golden_toy_preprocess():
    g, src, dst, et, *_ = toy()
    p = oracle.preprocess(g["V"], g["R"], src, dst, et)
    exp = g["preprocess"]
    for k in ["perm", "src_s", "seg", "row_ptr", "pos", "et_slot", "cnt"]:
        assert getattr(p, k).tolist() == exp[k], k


def test_golden_toy_rgcn():
    g, src, dst, et, X, W, A = toy()
    Y = oracle.rgcn_forward(g["V"], g["R"], src, dst, et, X, W)
    assert Y.tolist() == g["rgcn"]["Y"]  # exact: all values are small dyadic rationals


def test_golden_toy_rgat():
    g, src, dst, et, X, W, A = toy()
    Y, lse, alpha = oracle.rgat_forward(g["V"], g["R"], src, dst, et, X, W, A, slope=g["slope"], want_alpha=True)
    s = g["rgat"]["s"]
    z = np.array(g["rgat"]["zi"], float)
    den = math.exp(s[0]) + math.exp(s[1]) + math.exp(s[2])
    a_hand = [math.exp(s[0]) / den, math.exp(s[1]) / den, math.exp(s[2]) / den, 1.0]
    np.testing.assert_allclose(alpha, a_hand, rtol=1e-13, atol=0)
    np.testing.assert_allclose(alpha, g["rgat"]["alpha_12digits"], rtol=0, atol=6e-13)
    Y2 = a_hand[0] * z[0] + a_hand[1] * z[1] + a_hand[2] * z[2]
    np.testing.assert_allclose(Y[2], Y2, rtol=1e-13)
    np.testing.assert_allclose(Y, g["rgat"]["Y_12digits"], rtol=0, atol=6e-12)
    assert Y[0].tolist() == z[3].tolist()  # single in-edge: alpha = 1 exactly
    assert lse[1] == -math.inf and Y[1].tolist() == [0.0, 0.0]
    np.testing.assert_allclose(lse[2], math.log(den), rtol=1e-14)


# ---------------------------------------------------------------- P1 preprocessing
def _brute_preprocess(V, R, src, dst, et, v0, v1):
    own = [e for e in range(len(src)) if v0 <= dst[e] < v1]
    perm = sorted(own, key=lambda e: (int(et[e]), int(dst[e]), e))  # Python's sort on a total key
    seg = [sum(1 for e in own if et[e] < r) for r in range(R + 1)]
    rows = [[p for p, e in enumerate(perm) if dst[e] == v] for v in range(v0, v1)]
    row_ptr = [0]
    for r in rows:
        row_ptr.append(row_ptr[-1] + len(r))
    pos = [p for r in rows for p in r]
    cnt = [sum(1 for f in own if et[f] == et[e] and dst[f] == dst[e]) for e in perm]
    return perm, seg, row_ptr, pos, cnt


@pytest.mark.parametrize("seed,V,E,R,shard", [(0, 7, 30, 3, None), (1, 20, 200, 5, None), (2, 1, 10, 2, None),
                                              (3, 12, 0, 3, None), (4, 15, 120, 4, (5, 11)), (5, 9, 60, 1, None)])
def test_preprocess_bruteforce(seed, V, E, R, shard):
    g = synth.random_graph(V, E, R, seed)
    v0, v1 = shard or (0, V)
    p = oracle.preprocess(V, R, g.src, g.dst, g.etype, v0, v1)
    perm, seg, row_ptr, pos, cnt = _brute_preprocess(V, R, g.src, g.dst, g.etype, v0, v1)
    assert p.perm.tolist() == perm
    assert p.seg.tolist() == seg
    assert p.row_ptr.tolist() == row_ptr
    assert p.pos.tolist() == pos
    assert p.cnt.tolist() == cnt
    assert p.src_s.tolist() == [int(g.src[e]) for e in perm]
    assert p.et_slot.tolist() == [int(g.etype[perm[q]]) for q in pos]
    # invariants: multiset round trip; keys nondecreasing; rows hold their dst
    trip = sorted((int(g.src[e]), int(g.dst[e]), int(g.etype[e])) for e in p.perm)
    assert trip == sorted((int(g.src[e]), int(g.dst[e]), int(g.etype[e])) for e in range(E) if v0 <= g.dst[e] < v1)
    keys = [(int(g.etype[e]), int(g.dst[e])) for e in p.perm]
    assert keys == sorted(keys)
    for i in range(v1 - v0):
        for q in range(p.row_ptr[i], p.row_ptr[i + 1]):
            assert g.dst[p.perm[p.pos[q]]] == v0 + i


def test_preprocess_range_error_reports_smallest_edge():
    src = np.array([0, 1, 5, 0, 9], np.int32)
    dst = np.array([1, 0, 0, 7, 0], np.int32)
    et = np.array([0, 0, 0, 0, 3], np.int32)
    with pytest.raises(oracle.RangeError) as ei:
        oracle.preprocess(4, 2, src, dst, et)
    assert ei.value.edge_id == 2


# ---------------------------------------------------------------- P2/P3/P11 RGCN closed forms
def _dense_adj(V, R, src, dst, et, norm, edge_norm=None):
    """A_hat[r] [V,V] with A_hat[r][v,u] = sum over edges u->v of relation r of the norm factor."""
    Ah = np.zeros((R, V, V))
    cnt = np.zeros((R, V))
    np.add.at(cnt, (et, dst), 1.0)
    for e in range(len(src)):
        if norm == oracle.NORM_REL_INDEG:
            f = 1.0 / cnt[et[e], dst[e]]
        elif norm == oracle.NORM_NONE:
            f = 1.0
        else:
            f = edge_norm[e]
        Ah[et[e], dst[e], src[e]] += f
    return Ah


@pytest.mark.parametrize("norm", [oracle.NORM_REL_INDEG, oracle.NORM_NONE, oracle.NORM_EDGE])
@pytest.mark.parametrize("w0", [False, True])
def test_rgcn_dense_sum(norm, w0):
    V, E, R, K, N = 13, 70, 4, 5, 3
    g = synth.random_graph(V, E, R, seed=11)
    t = synth.make_tensors(V, R, K, N)
    en = np.random.default_rng(7).uniform(0.1, 1.0, E)
    Ah = _dense_adj(V, R, g.src, g.dst, g.etype, norm, en)
    X, W = t.X.astype(float), t.W.astype(float)
    ref = sum(Ah[r] @ X @ W[r] for r in range(R)) + (X @ t.W0.astype(float) if w0 else 0.0)
    Y = oracle.rgcn_forward(V, R, g.src, g.dst, g.etype, X, W, t.W0 if w0 else None, norm=norm, edge_norm=en)
    np.testing.assert_allclose(Y, ref, rtol=1e-12, atol=1e-13)


def test_rgcn_identity_is_spmm():
    scipy_sparse = pytest.importorskip("scipy.sparse")
    V, E, K = 25, 140, 6
    g = synth.random_graph(V, E, 1, seed=3)
    X = np.random.default_rng(1).standard_normal((V, K))
    Asp = scipy_sparse.coo_matrix((np.ones(E), (g.dst, g.src)), shape=(V, V)).tocsr()
    Y = oracle.rgcn_forward(V, 1, g.src, g.dst, g.etype, X, np.eye(K)[None], norm=oracle.NORM_NONE)
    np.testing.assert_allclose(Y, Asp @ X, rtol=1e-13, atol=1e-13)


@pytest.mark.parametrize("norm", [oracle.NORM_REL_INDEG, oracle.NORM_EDGE])
def test_rgcn_dw_closed_form(norm):
    V, E, R, K, N = 11, 60, 3, 4, 5
    g = synth.random_graph(V, E, R, seed=5)
    t = synth.make_tensors(V, R, K, N)
    en = np.random.default_rng(2).uniform(0.1, 1.0, E)
    Ah = _dense_adj(V, R, g.src, g.dst, g.etype, norm, en)
    X, G = t.X.astype(float), t.dY.astype(float)
    dW, dW0 = oracle.rgcn_backward(V, R, g.src, g.dst, g.etype, X, G, K, N, norm=norm, edge_norm=en, with_w0=True)
    for r in range(R):
        np.testing.assert_allclose(dW[r], (Ah[r] @ X).T @ G, rtol=1e-12, atol=1e-13)
    np.testing.assert_allclose(dW0, X.T @ G, rtol=1e-12, atol=1e-13)


# ---------------------------------------------------------------- P4-P7 RGAT special cases
def test_rgat_single_in_edge_alpha_one():
    V, K, N = 5, 4, 3
    src = np.array([3, 0, 2], np.int32); dst = np.array([1, 4, 0], np.int32); et = np.array([1, 0, 1], np.int32)
    t = synth.make_tensors(V, 2, K, N)
    Y, lse, al = oracle.rgat_forward(V, 2, src, dst, et, t.X, t.W, t.A, want_alpha=True)
    assert al.tolist() == [1.0, 1.0, 1.0]
    for e in range(3):
        np.testing.assert_allclose(Y[dst[e]], t.X[src[e]].astype(float) @ t.W[et[e]].astype(float), rtol=1e-14)


def test_rgat_star_identical_leaves_uniform():
    V, K, N, deg = 9, 4, 4, 8
    src = np.arange(1, 9, dtype=np.int32); dst = np.zeros(8, np.int32); et = np.zeros(8, np.int32)
    t = synth.make_tensors(V, 1, K, N)
    X = t.X.astype(float).copy(); X[1:] = X[1]
    _, _, al = oracle.rgat_forward(V, 1, src, dst, et, X, t.W, t.A, want_alpha=True)
    np.testing.assert_allclose(al, np.full(deg, 1.0 / deg), rtol=1e-14)


def test_rgat_zero_attention_is_mean_over_all_relations():
    V, E, R, K, N = 10, 80, 3, 4, 5
    g = synth.random_graph(V, E, R, seed=9)
    t = synth.make_tensors(V, R, K, N)
    Y, _, _ = oracle.rgat_forward(V, R, g.src, g.dst, g.etype, t.X, t.W, np.zeros_like(t.A))
    X, W = t.X.astype(float), t.W.astype(float)
    ref = np.zeros((V, N)); deg = np.bincount(g.dst, minlength=V)
    for e in range(E):
        ref[g.dst[e]] += X[g.src[e]] @ W[g.etype[e]] / deg[g.dst[e]]
    np.testing.assert_allclose(Y, ref, rtol=1e-13, atol=1e-14)


@pytest.mark.parametrize("a_scale", [1.0, 10.0])
def test_rgat_alpha_sums_to_one(a_scale):
    g = synth.make_graph(synth.get_config("mutag").scaled(50))
    t = synth.make_tensors(g.V, g.R, 8, 8, a_scale=a_scale)
    _, lse, al = oracle.rgat_forward(g.V, g.R, g.src, g.dst, g.etype, t.X, t.W, t.A,
                                     want_alpha=True)
    sums = np.zeros(g.V); np.add.at(sums, g.dst, al)
    deg = np.bincount(g.dst, minlength=g.V)
    np.testing.assert_allclose(sums[deg > 0], 1.0, atol=1e-12)
    assert np.all(np.isneginf(lse[deg == 0]))


def test_rgat_unstabilized_equals_stabilized():
    V, E, R, K, N = 12, 90, 3, 4, 4
    g = synth.random_graph(V, E, R, seed=4)
    t = synth.make_tensors(V, R, K, N)
    Y1, l1, a1 = oracle.rgat_forward(V, R, g.src, g.dst, g.etype, t.X, t.W, t.A, want_alpha=True)
    Y0, l0, a0 = oracle.rgat_forward(V, R, g.src, g.dst, g.etype, t.X, t.W, t.A, want_alpha=True, stabilize=False)
    np.testing.assert_allclose(Y0, Y1, rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(a0, a1, rtol=1e-12)


# ---------------------------------------------------------------- P8/P12 torch autograd
def _torch_rgat(V, src, dst, et, X, W, A, slope):
    """Independent vectorised fp64 torch RGAT: per-edge einsum + dense [V,E] masked log-softmax."""
    import torch
    s_, d_, e_ = (torch.as_tensor(a, dtype=torch.long) for a in (src, dst, et))
    zi = torch.einsum("ek,ekn->en", X[s_], W[e_])
    zj = torch.einsum("ek,ekn->en", X[d_], W[e_])
    pre = (A[e_, 0] * zi).sum(-1) + (A[e_, 1] * zj).sum(-1)
    s = torch.nn.functional.leaky_relu(pre, slope)
    mask = torch.zeros(V, len(src), dtype=torch.bool)
    mask[d_, torch.arange(len(src))] = True
    logits = torch.where(mask, s[None, :], torch.full_like(mask, -torch.inf, dtype=torch.float64))
    has = mask.any(1)
    alpha = torch.zeros_like(logits)
    alpha[has] = torch.softmax(logits[has], dim=1)
    return alpha @ zi


@pytest.mark.parametrize("slope", [0.2, 0.01])
def test_rgat_forward_backward_vs_torch_autograd(slope):
    torch = pytest.importorskip("torch")
    V, E, R, K, N = 9, 40, 3, 5, 4
    g = synth.random_graph(V, E, R, seed=21)
    t = synth.make_tensors(V, R, K, N)
    X = torch.tensor(t.X, dtype=torch.float64)
    W = torch.tensor(t.W, dtype=torch.float64, requires_grad=True)
    A = torch.tensor(t.A, dtype=torch.float64, requires_grad=True)
    G = torch.tensor(t.dY[:, :N], dtype=torch.float64)
    Yt = _torch_rgat(V, g.src, g.dst, g.etype, X, W, A, slope)
    (Yt * G).sum().backward()
    Y, _, _ = oracle.rgat_forward(V, R, g.src, g.dst, g.etype, t.X, t.W, t.A, slope=slope)
    np.testing.assert_allclose(Y, Yt.detach().numpy(), rtol=1e-12, atol=1e-14)
    dW, dA = oracle.rgat_backward(V, R, g.src, g.dst, g.etype, t.X, t.W, t.A, G.numpy(), slope=slope)
    np.testing.assert_allclose(dW, W.grad.numpy(), rtol=1e-11, atol=1e-13)
    np.testing.assert_allclose(dA, A.grad.numpy(), rtol=1e-11, atol=1e-13)


def test_rgat_r1_identity_is_gat():
    """R=1, W=I: single-head GAT with identity projection (P8); dense masked softmax in torch."""
    torch = pytest.importorskip("torch")
    V, E, K = 8, 30, 4
    g = synth.random_graph(V, E, 1, seed=8)
    X = np.random.default_rng(0).standard_normal((V, K))
    A = np.random.default_rng(1).standard_normal((1, 2, K))
    Xt = torch.tensor(X)
    el = Xt @ torch.tensor(A[0, 0]); er = Xt @ torch.tensor(A[0, 1])
    Y = np.zeros((V, K))
    for v in range(V):
        ins = np.nonzero(g.dst == v)[0]
        if len(ins):
            sc = torch.nn.functional.leaky_relu(el[g.src[ins]] + er[v], 0.2)
            Y[v] = (torch.softmax(sc, 0)[:, None] * Xt[g.src[ins]]).sum(0).numpy()
    Yo, _, _ = oracle.rgat_forward(V, 1, g.src, g.dst, g.etype, X, np.eye(K)[None], A)
    np.testing.assert_allclose(Yo, Y, rtol=1e-12, atol=1e-14)


# ---------------------------------------------------------------- P10 finite differences
def _fd(f, x, idx, h=1e-6):
    xp = x.copy(); xp[idx] += h
    xm = x.copy(); xm[idx] -= h
    return (f(xp) - f(xm)) / (2 * h)


def test_fd_gradients_rgat():
    V, E, R, K, N = 7, 25, 2, 3, 3
    g = synth.random_graph(V, E, R, seed=31)
    t = synth.make_tensors(V, R, K, N)
    X, W, A, G = (a.astype(float) for a in (t.X, t.W, t.A, t.dY[:, :N]))
    slope = 0.2

    def L(W_, A_):
        Y, _, _ = oracle.rgat_forward(V, R, g.src, g.dst, g.etype, X, W_, A_, slope=slope)
        return float((Y * G).sum())

    dW, dA = oracle.rgat_backward(V, R, g.src, g.dst, g.etype, X, W, A, G, slope=slope)
    rng = np.random.default_rng(0)
    for _ in range(12):
        idx = tuple(rng.integers(0, s) for s in W.shape)
        n = _fd(lambda w: L(w, A), W, idx)
        assert abs(dW[idx] - n) / max(abs(dW[idx]), abs(n), 1e-8) < 1e-4
        idx = tuple(rng.integers(0, s) for s in A.shape)
        n = _fd(lambda a: L(W, a), A, idx)
        assert abs(dA[idx] - n) / max(abs(dA[idx]), abs(n), 1e-8) < 1e-4


def test_fd_gradients_rgcn():
    V, E, R, K, N = 8, 30, 3, 3, 2
    g = synth.random_graph(V, E, R, seed=32)
    t = synth.make_tensors(V, R, K, N)
    X, W, W0, G = (a.astype(float) for a in (t.X, t.W, t.W0, t.dY[:, :N]))

    def L(W_, W0_):
        return float((oracle.rgcn_forward(V, R, g.src, g.dst, g.etype, X, W_, W0_) * G).sum())

    dW, dW0 = oracle.rgcn_backward(V, R, g.src, g.dst, g.etype, X, G, K, N, with_w0=True)
    for idx in [(0, 0, 0), (1, 2, 1), (2, 1, 0)]:
        n = _fd(lambda w: L(w, W0), W, idx)
        assert abs(dW[idx] - n) / max(abs(dW[idx]), abs(n), 1e-8) < 1e-4
    for idx in [(0, 0), (2, 1)]:
        n = _fd(lambda w0: L(W, w0), W0, idx)
        assert abs(dW0[idx] - n) / max(abs(dW0[idx]), abs(n), 1e-8) < 1e-4


# ---------------------------------------------------------------- P13 invariances, shard sums
def test_invariances():
    V, E, R, K, N = 14, 90, 4, 4, 4
    g = synth.random_graph(V, E, R, seed=41)
    t = synth.make_tensors(V, R, K, N)
    rng = np.random.default_rng(3)
    Y, _, _ = oracle.rgat_forward(V, R, g.src, g.dst, g.etype, t.X, t.W, t.A)
    # node relabel permutes Y
    pv = rng.permutation(V)
    inv = np.argsort(pv)
    Yn, _, _ = oracle.rgat_forward(V, R, pv[g.src], pv[g.dst], g.etype, t.X[inv], t.W, t.A)
    np.testing.assert_allclose(Yn[pv], Y, rtol=1e-12, atol=1e-14)
    # relation relabel with permuted W, A leaves Y unchanged
    pr = rng.permutation(R)
    Wr = np.empty_like(t.W); Wr[pr] = t.W
    Ar = np.empty_like(t.A); Ar[pr] = t.A
    Yr, _, _ = oracle.rgat_forward(V, R, g.src, g.dst, pr[g.etype], t.X, Wr, Ar)
    np.testing.assert_allclose(Yr, Y, rtol=1e-12, atol=1e-14)
    # COO order permutation
    pe = rng.permutation(E)
    Ye, _, _ = oracle.rgat_forward(V, R, g.src[pe], g.dst[pe], g.etype[pe], t.X, t.W, t.A)
    np.testing.assert_allclose(Ye, Y, rtol=1e-12, atol=1e-14)


def test_dst_shards_sum_to_full_gradient():
    V, E, R, K, N = 16, 120, 3, 4, 4
    g = synth.random_graph(V, E, R, seed=51)
    t = synth.make_tensors(V, R, K, N)
    G = t.dY[:, :N]
    dW, dA = oracle.rgat_backward(V, R, g.src, g.dst, g.etype, t.X, t.W, t.A, G)
    cuts = [0, 5, 9, 16]
    parts = [oracle.rgat_backward(V, R, g.src, g.dst, g.etype, t.X, t.W, t.A, G, v0=a, v1=b)
             for a, b in zip(cuts[:-1], cuts[1:])]
    np.testing.assert_allclose(sum(p[0] for p in parts), dW, rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(sum(p[1] for p in parts), dA, rtol=1e-12, atol=1e-14)
    # relation mask selects exactly that relation's slice
    dW1, dA1 = oracle.rgat_backward(V, R, g.src, g.dst, g.etype, t.X, t.W, t.A, G, rels=[1])
    np.testing.assert_allclose(dW1[1], dW[1], rtol=1e-12, atol=1e-14)
    assert not dW1[0].any() and not dW1[2].any()


# ---------------------------------------------------------------- compact materialisation
def test_golden_compact_toy():
    with open(os.path.join(os.path.dirname(__file__), "golden", "compact_toy.json")) as f:
        t = json.load(f)
    e = np.array(t["edges_src_dst_etype"])
    pre = oracle.preprocess(t["V"], t["R"], e[:, 0], e[:, 1], e[:, 2])
    c = oracle.compaction(t["R"], pre)
    assert pre.E_own == t["vanilla_rows"] and c.num_compact == t["compact_rows"]
    assert pre.perm.tolist() == t["perm"]
    assert c.crow_of_pos.tolist() == t["crow_of_pos"]
    assert c.csrc.tolist() == t["csrc"] and c.cseg.tolist() == t["cseg"]


@pytest.mark.parametrize("seed,V,E,R,shard", [(0, 50, 400, 3, False), (1, 300, 2000, 7, True), (2, 5, 0, 2, False),
                                              (3, 1, 30, 1, False)])
def test_compaction_bruteforce(seed, V, E, R, shard):
    rng = np.random.default_rng(seed)
    src = rng.integers(0, V, E); dst = rng.integers(0, V, E); et = rng.integers(0, R, E)
    v0, v1 = (V // 3, 2 * V // 3) if shard else (0, V)
    pre = oracle.preprocess(V, R, src, dst, et, v0, v1)
    c = oracle.compaction(R, pre)
    own = (dst >= v0) & (dst < v1)
    # U = number of distinct (etype, src) pairs of the owned edges, counted another way
    assert c.num_compact == np.unique(et[own].astype(np.int64) * V + src[own]).size
    # every position's compact row holds exactly its (etype, src)
    et_p = et[pre.perm]
    assert (c.csrc[c.crow_of_pos] == src[pre.perm]).all() and (c.crel[c.crow_of_pos] == et_p).all()
    # rows strictly increasing in (etype, src); cseg brackets each relation
    key = c.crel.astype(np.int64) * V + c.csrc
    assert (np.diff(key) > 0).all()
    for r in range(R):
        assert (c.crel[c.cseg[r]:c.cseg[r + 1]] == r).all()
    assert c.cseg[0] == 0 and c.cseg[R] == c.num_compact


# ---------------------------------------------------------------- dX (NEXT-2)
@pytest.mark.parametrize("slope", [0.2, 0.01])
def test_rgat_dx_vs_torch_autograd(slope):
    """oracle.rgat_dx equals the X-gradient of the independent torch RGAT (_torch_rgat)."""
    torch = pytest.importorskip("torch")
    V, E, R, K, N = 9, 40, 3, 5, 4
    g = synth.random_graph(V, E, R, seed=22)
    t = synth.make_tensors(V, R, K, N)
    X = torch.tensor(t.X, dtype=torch.float64, requires_grad=True)
    W = torch.tensor(t.W, dtype=torch.float64)
    A = torch.tensor(t.A, dtype=torch.float64)
    G = torch.tensor(t.dY[:, :N], dtype=torch.float64)
    (_torch_rgat(V, g.src, g.dst, g.etype, X, W, A, slope) * G).sum().backward()
    dX = oracle.rgat_dx(V, R, g.src, g.dst, g.etype, t.X, t.W, t.A, G.numpy(), slope=slope)
    np.testing.assert_allclose(dX, X.grad.numpy(), rtol=1e-11, atol=1e-13)


def test_fd_gradients_dx():
    V, E, R, K, N = 7, 25, 2, 3, 3
    g = synth.random_graph(V, E, R, seed=33)
    t = synth.make_tensors(V, R, K, N)
    X, W, W0, A, G = (a.astype(float) for a in (t.X, t.W, t.W0, t.A, t.dY[:, :N]))

    def Lgat(X_):
        Y, _, _ = oracle.rgat_forward(V, R, g.src, g.dst, g.etype, X_, W, A)
        return float((Y * G).sum())

    def Lgcn(X_):
        return float((oracle.rgcn_forward(V, R, g.src, g.dst, g.etype, X_, W, W0) * G).sum())

    dXa = oracle.rgat_dx(V, R, g.src, g.dst, g.etype, X, W, A, G)
    dXc = oracle.rgcn_dx(V, R, g.src, g.dst, g.etype, W, G, W0=W0)
    rng = np.random.default_rng(1)
    for _ in range(10):
        idx = tuple(rng.integers(0, s) for s in X.shape)
        n = _fd(Lgat, X, idx)
        assert abs(dXa[idx] - n) / max(abs(dXa[idx]), abs(n), 1e-8) < 1e-4
        n = _fd(Lgcn, X, idx)
        assert abs(dXc[idx] - n) / max(abs(dXc[idx]), abs(n), 1e-8) < 1e-4


@pytest.mark.parametrize("norm", [0, 1, 2])
def test_rgcn_dx_closed_form(norm):
    """dX = sum_r A_r^T G W_r^T + G W0^T with the dense normalised adjacency A_r (NumPy)."""
    V, E, R, K, N = 20, 150, 3, 4, 5
    g = synth.random_graph(V, E, R, seed=34)
    t = synth.make_tensors(V, R, K, N)
    en = np.random.default_rng(2).uniform(0.1, 1, E)
    G = t.dY[:, :N].astype(float)
    ref = G @ t.W0.astype(float).T
    for r in range(R):
        Ar = np.zeros((V, V))
        m = g.etype == r
        np.add.at(Ar, (g.dst[m], g.src[m]), en[m] if norm == 2 else 1.0)
        if norm == 0:
            c = np.bincount(g.dst[m], minlength=V).astype(float)
            Ar = Ar / np.maximum(c, 1)[:, None]
        ref += Ar.T @ G @ t.W[r].astype(float).T
    got = oracle.rgcn_dx(V, R, g.src, g.dst, g.etype, t.W, G, W0=t.W0, norm=norm,
                         edge_norm=en if norm == 2 else None)
    np.testing.assert_allclose(got, ref, rtol=1e-12, atol=1e-12)


def test_dx_dst_shards_sum_to_full():
    V, E, R, K, N = 30, 300, 4, 4, 4
    g = synth.random_graph(V, E, R, seed=35)
    t = synth.make_tensors(V, R, K, N)
    G = t.dY[:, :N]
    full = oracle.rgat_dx(V, R, g.src, g.dst, g.etype, t.X, t.W, t.A, G)
    parts = sum(oracle.rgat_dx(V, R, g.src, g.dst, g.etype, t.X, t.W, t.A, G, v0=a, v1=b)
                for a, b in [(0, 11), (11, 12), (12, 30)])
    np.testing.assert_allclose(parts, full, rtol=1e-12, atol=1e-13)


# ---------------------------------------------------------------- HGT (NEXT-3)
def _torch_hgt(V, src, dst, et, ntype, X, WK, WQ, WV, Wa, Wm):
    """Independent vectorised fp64 torch HGT: per-node typed linears, per-edge bilinear score,
    dense [V, E] masked softmax."""
    import torch
    s_, d_, e_ = (torch.as_tensor(a, dtype=torch.long) for a in (src, dst, et))
    nt = torch.as_tensor(ntype, dtype=torch.long)
    Kn = torch.einsum("vk,vkn->vn", X, WK[nt])
    Qn = torch.einsum("vk,vkn->vn", X, WQ[nt])
    Vn = torch.einsum("vk,vkn->vn", X, WV[nt])
    a = torch.einsum("em,emn,en->e", Kn[s_], Wa[e_], Qn[d_])
    msg = torch.einsum("em,emn->en", Vn[s_], Wm[e_])
    mask = torch.zeros(V, len(src), dtype=torch.bool)
    mask[d_, torch.arange(len(src))] = True
    logits = torch.where(mask, a[None, :], torch.full_like(mask, -torch.inf, dtype=torch.float64))
    has = mask.any(1)
    alpha = torch.zeros_like(logits)
    alpha[has] = torch.softmax(logits[has], dim=1)
    return alpha @ msg


def test_hgt_vs_torch():
    torch = pytest.importorskip("torch")
    V, E, R, T, K, N = 12, 60, 3, 2, 5, 4
    g = synth.random_graph(V, E, R, seed=51, T=T)
    t = synth.make_hgt_tensors(V, R, T, K, N)
    args = [torch.tensor(a, dtype=torch.float64) for a in (t.X, t.WK, t.WQ, t.WV, t.Wa, t.Wm)]
    ref = _torch_hgt(V, g.src, g.dst, g.etype, g.ntype, *args).numpy()
    Y, lse = oracle.hgt_forward(V, R, g.src, g.dst, g.etype, g.ntype, t.X, t.WK, t.WQ, t.WV, t.Wa, t.Wm)
    np.testing.assert_allclose(Y, ref, rtol=1e-12, atol=1e-14)
    deg = np.bincount(g.dst, minlength=V)
    assert np.isneginf(lse[deg == 0]).all() and np.isfinite(lse[deg > 0]).all()


def test_hgt_one_type_identity_is_dot_product_attention():
    """T = R = 1, W_a = W_m = I: graph-masked single-head dot-product attention softmax(Q K^T) V
    (torch.nn.functional.scaled_dot_product_attention with scale 1 and the adjacency as mask)."""
    torch = pytest.importorskip("torch")
    V, E, K, N = 10, 45, 4, 3
    g = synth.random_graph(V, E, 1, seed=52)
    t = synth.make_hgt_tensors(V, 1, 1, K, N)
    I = np.eye(N)[None]
    Y, _ = oracle.hgt_forward(V, 1, g.src, g.dst, g.etype, np.zeros(V, np.int32), t.X, t.WK, t.WQ, t.WV, I, I)
    X = torch.tensor(t.X, dtype=torch.float64)
    Q, Kt, Vt = X @ torch.tensor(t.WQ[0], dtype=torch.float64), X @ torch.tensor(t.WK[0], dtype=torch.float64), \
        X @ torch.tensor(t.WV[0], dtype=torch.float64)
    cnt = np.zeros((V, V))
    np.add.at(cnt, (g.dst, g.src), 1.0)  # multi-edges count twice in the softmax
    has = cnt.sum(1) > 0
    bias = torch.tensor(np.where(cnt > 0, np.log(np.maximum(cnt, 1)), -np.inf))
    out = torch.nn.functional.scaled_dot_product_attention(Q[has][None], Kt[None], Vt[None],
                                                           attn_mask=bias[has][None], scale=1.0)[0]
    np.testing.assert_allclose(Y[has], out.numpy(), rtol=1e-12, atol=1e-13)
    assert not Y[~has].any()


def test_hgt_softmax_weights_sum_to_one():
    """Messages identically 1 (V s = const, W_m chosen so m = 1): Y_t = sum alpha = 1 on rows with in-edges."""
    V, E, R, T, K, N = 15, 80, 3, 2, 4, 4
    g = synth.random_graph(V, E, R, seed=53, T=T)
    t = synth.make_hgt_tensors(V, R, T, K, N)
    X = t.X.copy(); X[:, 0] = 1.0
    WV = np.zeros_like(t.WV); WV[:, 0, 0] = 1.0          # v = e_0 for every node
    Wm = np.zeros_like(t.Wm); Wm[:, 0, :] = 1.0          # m = v W_m = all-ones
    Y, _ = oracle.hgt_forward(V, R, g.src, g.dst, g.etype, g.ntype, X, t.WK * 5, t.WQ * 5, WV, t.Wa, Wm)
    deg = np.bincount(g.dst, minlength=V)
    np.testing.assert_allclose(Y[deg > 0], 1.0, atol=1e-12)


def test_hgt_backward_vs_torch_autograd():
    torch = pytest.importorskip("torch")
    V, E, R, T, K, N = 12, 60, 3, 2, 5, 4
    g = synth.random_graph(V, E, R, seed=54, T=T)
    t = synth.make_hgt_tensors(V, R, T, K, N)
    X = torch.tensor(t.X, dtype=torch.float64)
    Ws = [torch.tensor(a, dtype=torch.float64, requires_grad=True) for a in (t.WK, t.WQ, t.WV, t.Wa, t.Wm)]
    G = torch.tensor(t.dY[:, :N], dtype=torch.float64)
    (_torch_hgt(V, g.src, g.dst, g.etype, g.ntype, X, *Ws) * G).sum().backward()
    got = oracle.hgt_backward(V, R, g.src, g.dst, g.etype, g.ntype, t.X, t.WK, t.WQ, t.WV, t.Wa, t.Wm, G.numpy())
    for name, a, w in zip(["dWK", "dWQ", "dWV", "dWa", "dWm"], got, Ws):
        np.testing.assert_allclose(a, w.grad.numpy(), rtol=1e-11, atol=1e-13, err_msg=name)


def test_hgt_backward_fd_and_shards():
    V, E, R, T, K, N = 8, 30, 2, 2, 3, 3
    g = synth.random_graph(V, E, R, seed=55, T=T)
    t = synth.make_hgt_tensors(V, R, T, K, N)
    Wl = [a.astype(float) for a in (t.WK, t.WQ, t.WV, t.Wa, t.Wm)]
    G = t.dY[:, :N].astype(float)

    def L(ws):
        Y, _ = oracle.hgt_forward(V, R, g.src, g.dst, g.etype, g.ntype, t.X, *ws)
        return float((Y * G).sum())

    got = oracle.hgt_backward(V, R, g.src, g.dst, g.etype, g.ntype, t.X, *Wl, G)
    rng = np.random.default_rng(2)
    for wi in range(5):
        for _ in range(3):
            idx = tuple(rng.integers(0, s) for s in Wl[wi].shape)
            n = _fd(lambda w: L(Wl[:wi] + [w] + Wl[wi + 1:]), Wl[wi], idx)
            assert abs(got[wi][idx] - n) / max(abs(got[wi][idx]), abs(n), 1e-8) < 1e-4, (wi, idx)
    parts = [oracle.hgt_backward(V, R, g.src, g.dst, g.etype, g.ntype, t.X, *Wl, G, v0=a, v1=b)
             for a, b in [(0, 3), (3, 8)]]
    for wi in range(5):
        np.testing.assert_allclose(parts[0][wi] + parts[1][wi], got[wi], rtol=1e-12, atol=1e-13)
