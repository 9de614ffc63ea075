"""Seeded synthetic heterographs shaped like the paper's datasets.

Shapes: PAPER.md tab:datasets and BASELINE.json `configs`.
Degree laws and calibration: SURVEY.md §8(d) (AM-shaped a_rel=1.0, a_src=0.6,
a_dst=0.8 gives a (etype,src) compaction ratio close to the 57% the paper
prints for AM).

Recipe (NumPy PCG64, one stream per seed):
  * node types: contiguous id ranges; sizes Zipf(1.0) split of V (floor 100
    per type) unless explicit sizes are given (ogbn-mag);
  * relation sizes E_r ~ Zipf(a_rel) with min 1, the largest relation absorbs
    the rounding so sum E_r = E exactly; sizes are assigned to relation ids in
    a seeded random order;
  * each relation's (src type, dst type) signature is drawn uniformly (or given);
  * src / dst ids: Zipf(a_src) / Zipf(a_dst) over node ranks of the type,
    mapped through a seeded per-type permutation, so hubs are scattered in id
    space;
  * multi-edges and self-edges are kept; the final COO order is a seeded
    shuffle (the input is NOT presorted).
Tensors: X ~ U(-1,1); W_r ~ Glorot U(+-sqrt(6/(K+N))); A[r] ~ U(+-sqrt(6/(2N+1)));
dY ~ U(-1,1); all fp32.

No layer arithmetic lives here.
"""
from __future__ import annotations

import dataclasses
from typing import Optional, Sequence

import numpy as np

GRAPH_SEED, X_SEED, W_SEED, A_SEED, DY_SEED, LABEL_SEED = 0, 1, 2, 3, 4, 5


@dataclasses.dataclass
class GraphConfig:
    name: str
    V: int
    E: int
    R: int
    T: int
    K: int
    N: int
    a_rel: float = 1.0
    a_src: float = 0.6
    a_dst: float = 0.8
    type_sizes: Optional[Sequence[int]] = None
    # optional explicit relations: list of (src_type, dst_type, E_r, a_dst or None)
    relations: Optional[Sequence[tuple]] = None
    prec: str = "bf16"
    model: str = "rgat"
    note: str = ""

    def scaled(self, factor: float, name: Optional[str] = None) -> "GraphConfig":
        """Same recipe with V and E divided by `factor` (parity-test sizes)."""
        V = max(int(self.V / factor), 8)
        E = max(int(self.E / factor), 1)
        ts = None
        if self.type_sizes is not None:
            ts = [max(int(s / factor), 4) for s in self.type_sizes]
            V = int(sum(ts))
        rels = None
        if self.relations is not None:
            rels = [(s, d, max(int(e / factor), 1), a) for (s, d, e, a) in self.relations]
            E = int(sum(r[2] for r in rels))
        R = self.R
        return dataclasses.replace(self, name=name or f"{self.name}/{factor:g}", V=V, E=E,
                                   R=R, type_sizes=ts, relations=rels)


_MAG_TYPES = [1134649, 736389, 8740, 59965]  # author, paper, institution, field (sum = 1,939,743)
_MAG_RELS = [  # (src type, dst type, E_r, a_dst override)
    (0, 2, 1043998, None),   # author -> institution
    (0, 1, 7145660, None),   # author -> paper
    (1, 1, 5416271, None),   # paper  -> paper
    (1, 3, 7505078, 1.0),    # paper  -> field (field hubs)
]

CONFIGS = {
    # BASELINE.json configs[0]: AIFB-shaped, RGCN fwd, d=32, fp32
    "aifb": GraphConfig("aifb", V=7262, E=48810, R=45, T=7, K=32, N=32, prec="f32", model="rgcn"),
    # configs[1]: MUTAG / BGS shaped, RGCN and RGAT fwd+bwd, d=64
    "mutag": GraphConfig("mutag", V=27163, E=148100, R=23, T=5, K=64, N=64, model="rgat"),
    "bgs": GraphConfig("bgs", V=94806, E=672900, R=103, T=27, K=64, N=64, model="rgat"),
    # configs[2]: AM-shaped, RGAT fwd+bwd, d=64, bf16 typed GEMM
    "am": GraphConfig("am", V=1885136, E=5668682, R=133, T=7, K=64, N=64, model="rgat"),
    # configs[3]: ogbn-mag shaped, RGAT d=128, dst-partitioned 1/2/4/8
    "mag": GraphConfig("mag", V=sum(_MAG_TYPES), E=sum(r[2] for r in _MAG_RELS), R=4, T=4,
                       K=128, N=128, type_sizes=_MAG_TYPES, relations=_MAG_RELS, model="rgat"),
    # configs[4]: ogbl-wikikg2 shaped, 535 skewed relations, RGCN d=64
    "wikikg2": GraphConfig("wikikg2", V=2500604, E=16109182, R=535, T=1, K=64, N=64,
                           a_rel=1.5, a_src=0.7, a_dst=0.8, model="rgcn"),
}


def get_config(name: str) -> GraphConfig:
    if "/" in name:  # "am/100" = AM recipe scaled down 100x
        base, f = name.split("/")
        return CONFIGS[base].scaled(float(f))
    return CONFIGS[name]


@dataclasses.dataclass
class HeteroGraph:
    V: int
    R: int
    T: int
    src: np.ndarray    # int32 [E]
    dst: np.ndarray    # int32 [E]
    etype: np.ndarray  # int32 [E]
    ntype: np.ndarray  # int32 [V]
    name: str = ""

    @property
    def E(self) -> int:
        return int(self.src.shape[0])


@dataclasses.dataclass
class LayerTensors:
    X: np.ndarray   # fp32 [V, K]
    W: np.ndarray   # fp32 [R, K, N]
    A: np.ndarray   # fp32 [R, 2, N]
    W0: np.ndarray  # fp32 [K, N]
    dY: np.ndarray  # fp32 [V, N]


def _zipf_sizes(total: int, parts: int, a: float, floor: int) -> np.ndarray:
    w = 1.0 / np.power(np.arange(1, parts + 1, dtype=np.float64), a)
    sizes = np.maximum(np.floor(w / w.sum() * total).astype(np.int64), floor)
    sizes[0] += total - sizes.sum()  # the largest absorbs the rounding
    if sizes[0] < floor:
        raise ValueError("total too small for the floor")
    return sizes


def _zipf_ranks(rng: np.random.Generator, n: int, a: float, size: int, cache: dict) -> np.ndarray:
    if n == 1:
        return np.zeros(size, dtype=np.int64)
    key = (n, a)
    cdf = cache.get(key)
    if cdf is None:
        w = 1.0 / np.power(np.arange(1, n + 1, dtype=np.float64), a)
        cdf = np.cumsum(w)
        cdf /= cdf[-1]
        cache[key] = cdf
    u = rng.random(size)
    return np.minimum(np.searchsorted(cdf, u, side="right"), n - 1)


def make_graph(cfg: GraphConfig, seed: int = GRAPH_SEED) -> HeteroGraph:
    rng = np.random.Generator(np.random.PCG64(seed))
    T, R, E = cfg.T, cfg.R, cfg.E
    if cfg.type_sizes is not None:
        tsz = np.asarray(cfg.type_sizes, dtype=np.int64)
    else:
        tsz = _zipf_sizes(cfg.V, T, 1.0, min(100, cfg.V // T))
    V = int(tsz.sum())
    toff = np.concatenate([[0], np.cumsum(tsz)])
    tperm = [rng.permutation(int(n)) for n in tsz]
    ntype = np.repeat(np.arange(T, dtype=np.int32), tsz)

    if cfg.relations is not None:
        rels = list(cfg.relations)
        R = len(rels)
    else:
        esz = _zipf_sizes(E, R, cfg.a_rel, 1)
        order = rng.permutation(R)  # relation id -> size rank
        sig = rng.integers(0, T, size=(R, 2))
        rels = [(int(sig[r, 0]), int(sig[r, 1]), int(esz[order[r]]), None) for r in range(R)]
    cache: dict = {}
    srcs, dsts, ets = [], [], []
    for r, (st, dt, er, adst) in enumerate(rels):
        a_d = cfg.a_dst if adst is None else adst
        su = _zipf_ranks(rng, int(tsz[st]), cfg.a_src, er, cache)
        du = _zipf_ranks(rng, int(tsz[dt]), a_d, er, cache)
        srcs.append(toff[st] + tperm[st][su])
        dsts.append(toff[dt] + tperm[dt][du])
        ets.append(np.full(er, r, dtype=np.int64))
    src = np.concatenate(srcs)
    dst = np.concatenate(dsts)
    et = np.concatenate(ets)
    shuf = rng.permutation(src.shape[0])
    return HeteroGraph(V=V, R=R, T=T, src=src[shuf].astype(np.int32), dst=dst[shuf].astype(np.int32),
                       etype=et[shuf].astype(np.int32), ntype=ntype, name=cfg.name)


def random_graph(V: int, E: int, R: int, seed: int = 0, T: int = 1) -> HeteroGraph:
    """Uniform random multigraph (tiny test graphs)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return HeteroGraph(V=V, R=R, T=T,
                       src=rng.integers(0, V, E).astype(np.int32),
                       dst=rng.integers(0, V, E).astype(np.int32),
                       etype=rng.integers(0, R, E).astype(np.int32),
                       ntype=rng.integers(0, T, V).astype(np.int32), name=f"rand{V}x{E}x{R}")


def make_tensors(V: int, R: int, K: int, N: int, seeds=(X_SEED, W_SEED, A_SEED, DY_SEED),
                 a_scale: float = 1.0) -> LayerTensors:
    xs, ws, as_, dys = seeds
    rx = np.random.Generator(np.random.PCG64(xs))
    rw = np.random.Generator(np.random.PCG64(ws))
    ra = np.random.Generator(np.random.PCG64(as_))
    rd = np.random.Generator(np.random.PCG64(dys))
    X = rx.uniform(-1.0, 1.0, size=(V, K)).astype(np.float32)
    gw = np.sqrt(6.0 / (K + N))
    W = rw.uniform(-gw, gw, size=(R, K, N)).astype(np.float32)
    W0 = rw.uniform(-gw, gw, size=(K, N)).astype(np.float32)
    ga = np.sqrt(6.0 / (2 * N + 1)) * a_scale
    A = ra.uniform(-ga, ga, size=(R, 2, N)).astype(np.float32)
    dY = rd.uniform(-1.0, 1.0, size=(V, N)).astype(np.float32)
    return LayerTensors(X=X, W=W, A=A, W0=W0, dY=dY)


@dataclasses.dataclass
class HgtTensors:
    X: np.ndarray    # fp32 [V, K]
    WK: np.ndarray   # fp32 [T, K, N]  node-typed key linear
    WQ: np.ndarray   # fp32 [T, K, N]  node-typed query linear
    WV: np.ndarray   # fp32 [T, K, N]  node-typed value linear
    Wa: np.ndarray   # fp32 [R, N, N]  relation attention matrix W_{a,r}
    Wm: np.ndarray   # fp32 [R, N, N]  relation message matrix W_{m,r}
    dY: np.ndarray   # fp32 [V, N]


def make_hgt_tensors(V: int, R: int, T: int, K: int, N: int, seeds=(X_SEED, W_SEED, A_SEED, DY_SEED)) -> HgtTensors:
    """Seeded HGT layer inputs (NEXT-3): U(-1,1) features, Glorot-uniform weights."""
    xs, ws, as_, dys = seeds
    rx = np.random.Generator(np.random.PCG64(xs))
    rw = np.random.Generator(np.random.PCG64(ws))
    ra = np.random.Generator(np.random.PCG64(as_))
    rd = np.random.Generator(np.random.PCG64(dys))
    X = rx.uniform(-1.0, 1.0, size=(V, K)).astype(np.float32)
    g1 = np.sqrt(6.0 / (K + N))
    WK, WQ, WV = (rw.uniform(-g1, g1, size=(T, K, N)).astype(np.float32) for _ in range(3))
    g2 = np.sqrt(6.0 / (2 * N))
    Wa = ra.uniform(-g2, g2, size=(R, N, N)).astype(np.float32)
    Wm = ra.uniform(-g2, g2, size=(R, N, N)).astype(np.float32)
    dY = rd.uniform(-1.0, 1.0, size=(V, N)).astype(np.float32)
    return HgtTensors(X=X, WK=WK, WQ=WQ, WV=WV, Wa=Wa, Wm=Wm, dY=dY)
