"""The RGAT backward with the messages recomputed in TMEM (csrc/bwd_tm.cu) against the fp64 oracle.

Both backward kernels of the bf16 layer run on every case: RGNN_BWD_TM=1 forces the tensor-core
message-recompute kernel, RGNN_BWD_TM=0 the fused kernel (bwd_fused_tc.cu); the default picks by the
mean (etype, dst) run length.  Cases cover every (d_in, d_out) in {64, 128}^2, long runs (a few
destinations), short runs whose count per 128-position stage exceeds the kernel's bf16 run-row
buffer (the fp32 fallback rows), hub rows split across stages and chunks, a destination-range
shard, compact and vanilla Z rows, dX (the (alpha, dpre) side output), and bit-determinism.
"""
import numpy as np
import pytest

import oracle
import synth
from parity import assert_close, run_gpu, run_oracle

pytestmark = pytest.mark.gpu


def _graphs():
    return {
        "long-runs": synth.random_graph(160, 24000, 3, seed=11),      # ~50 positions per (etype, dst) run
        "mag/100": synth.make_graph(synth.get_config("mag").scaled(100)),
        "am/60": synth.make_graph(synth.get_config("am").scaled(60)),  # runs of ~2: > CAP runs per stage
        "mutag/4": synth.make_graph(synth.get_config("mutag").scaled(4)),
    }


GRAPHS = _graphs()


def _run(m, monkeypatch, g, t, tm, **kw):
    monkeypatch.setenv("RGNN_BWD_TM", "1" if tm else "0")
    return run_gpu(m, g, t, "rgat", "bf16", **kw)


def _check(gpu, ref, what):
    assert_close(gpu["Y"], ref["Y"], "bf16", f"{what} Y")
    assert_close(gpu["dW"], ref["dW"], "bf16", f"{what} dW", per_slice=True)
    assert_close(gpu["dA"], ref["dA"], "bf16", f"{what} dA", per_slice=True)


@pytest.mark.parametrize("tm", [1, 0], ids=["tm", "fused"])
@pytest.mark.parametrize("kn", [(64, 64), (128, 128), (64, 128), (128, 64)], ids=lambda kn: f"{kn[0]}x{kn[1]}")
@pytest.mark.parametrize("name", list(GRAPHS))
def test_bwd_kernels_vs_oracle(rgnn, monkeypatch, name, kn, tm):
    g = GRAPHS[name]
    t = synth.make_tensors(g.V, g.R, *kn)
    mat = "auto" if name == "mag/100" else "vanilla"
    gpu = _run(rgnn, monkeypatch, g, t, tm, materialization=mat)
    ref = run_oracle(oracle, g, t, "rgat", prec="bf16")
    _check(gpu, ref, f"{name} {kn} tm={tm}")


@pytest.mark.parametrize("tm", [1, 0], ids=["tm", "fused"])
def test_bwd_tm_shard_and_split_rows(rgnn, monkeypatch, tm):
    g = GRAPHS["mag/100"]
    t = synth.make_tensors(g.V, g.R, 128, 128)
    rng = (g.V // 5, (4 * g.V) // 5)
    gpu = _run(rgnn, monkeypatch, g, t, tm, dst_range=rng, split_cap=64, materialization="compact")
    ref = run_oracle(oracle, g, t, "rgat", prec="bf16", dst_range=rng)
    _check(gpu, ref, f"shard tm={tm}")


@pytest.mark.parametrize("name", ["long-runs", "am/60"])
def test_bwd_tm_dx(rgnn, monkeypatch, name):
    """dX reads the kernel's (alpha, dpre) per position."""
    g = GRAPHS[name]
    t = synth.make_tensors(g.V, g.R, 64, 64)
    gpu = _run(rgnn, monkeypatch, g, t, 1, want_dx=True)
    ref = run_oracle(oracle, g, t, "rgat", prec="bf16", want_dx=True)
    _check(gpu, ref, f"{name} dx")
    assert_close(gpu["dX"], ref["dX"], "bf16", f"{name} dX")


def test_bwd_tm_deterministic(rgnn, monkeypatch):
    g = GRAPHS["mag/100"]
    t = synth.make_tensors(g.V, g.R, 128, 128)
    a = _run(rgnn, monkeypatch, g, t, 1, materialization="auto")
    b = _run(rgnn, monkeypatch, g, t, 1, materialization="auto")
    for k in ("dW", "dA"):
        np.testing.assert_array_equal(a[k], b[k], err_msg=k)


def test_bwd_tm_matches_fused_kernel(rgnn, monkeypatch):
    """The two kernels compute the same gradients (different rounding points only)."""
    g = GRAPHS["long-runs"]
    t = synth.make_tensors(g.V, g.R, 128, 128)
    a = _run(rgnn, monkeypatch, g, t, 1)
    b = _run(rgnn, monkeypatch, g, t, 0)
    for k in ("dW", "dA"):
        rel = np.linalg.norm(a[k] - b[k]) / np.linalg.norm(b[k])
        assert rel < 1e-2, (k, rel)
