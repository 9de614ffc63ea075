"""Kernel-level GPU checks: the tcgen05 typed GEMM's Z and s_src (read from the
`saved` buffer, layout of layer.cu SavedLayout) against a NumPy GEMM of the same
bf16 operands, for every supported (d_in, d_out) and ragged segment tails."""
import numpy as np
import pytest

import synth
from parity import bf16_round

pytestmark = pytest.mark.gpu


def _align(x, a=256):
    return (x + a - 1) // a * a


@pytest.mark.parametrize("K,N", [(32, 32), (64, 64), (128, 128), (64, 128), (128, 64), (32, 128), (128, 32), (64, 32),
                                 (32, 64)])
def test_tc_gemm_matches_numpy(rgnn, K, N):
    import torch
    g = synth.random_graph(3000, 20000, 9, seed=K + N)
    t = synth.make_tensors(g.V, g.R, K, N)
    G = rgnn.Graph(g.V, g.src, g.dst, g.etype, g.R)
    X = torch.from_numpy(t.X).cuda().to(torch.bfloat16)
    _, ws = rgnn.rgat_forward(G, X, torch.from_numpy(t.W).cuda(), torch.from_numpy(t.A).cuda(), prec="bf16")
    torch.cuda.synchronize()
    E = G.E_own
    arr = {k: v.cpu().numpy() for k, v in G.arrays().items()}
    Z = ws.saved[:E * N * 2].view(torch.bfloat16).float().cpu().numpy().reshape(E, N)
    off = _align(E * N * 2)
    s_src = ws.saved[off:off + E * 4].view(torch.float32).cpu().numpy()
    Xb, Wb = bf16_round(t.X).astype(np.float64), bf16_round(t.W).astype(np.float64)
    r_of_p = np.repeat(np.arange(g.R), np.diff(arr["seg"]))
    ref = np.einsum("pk,pkn->pn", Xb[arr["src_s"]], Wb[r_of_p])
    np.testing.assert_allclose(Z, ref, rtol=8e-3, atol=8e-3 * np.abs(ref).max())
    sref = np.einsum("pn,pn->p", ref, t.A[r_of_p, 0].astype(np.float64))
    np.testing.assert_allclose(s_src, sref, rtol=1e-4, atol=1e-4 * np.abs(sref).max())
