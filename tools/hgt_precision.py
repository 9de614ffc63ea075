"""Worst ratio of |GPU - oracle| to reading O19's bf16 bound (0.02 rms(slice) + 0.02 |ref|) for each
HGT gradient on three dst-range shards of a BGS-shaped graph (run on the GPU box):
    python tools/hgt_precision.py            (RGNN_DISABLE_TCGEN05=1 for the SIMT kernels)
Used to choose the HGT precision layout (O23)."""
import sys, os; sys.path.insert(0,'tests'); sys.path.insert(0,'.')
import numpy as np, synth
import paper_2301_06284_b200 as rgnn
import test_gpu_hgt as T
from parity import TOL
g = synth.make_graph(synth.get_config("bgs").scaled(10))
t = synth.make_hgt_tensors(g.V, g.R, g.T, 64, 64)
indeg = np.r_[0, np.cumsum(np.bincount(g.dst, minlength=g.V))]
b = rgnn.partition_dst(indeg, 3)
for k in range(3):
    rng = (int(b[k]), int(b[k + 1]))
    gs = T._run_bwd(rgnn, g, t, "bf16", dst_range=rng)
    ref = T._ref_bwd(g, t, "bf16", rng)
    out=[]
    for name, a, r in zip(T.GRAD_NAMES, gs, ref):
        rms = np.sqrt(np.mean(r*r, axis=(1,2), keepdims=True))
        ratio = np.max((np.abs(a-r)) / (0.02*rms + 0.02*np.abs(r) + 1e-30))
        out.append(f"{name} {ratio:.2f}")
    print(os.environ.get("RGNN_DISABLE_TCGEN05","tc"), "shard", k, " ".join(out), flush=True)
