"""compute-sanitizer over the hot path's mbarrier / TMEM / TMA pipelines (tools/sanitize_case.py).

memcheck (out-of-bounds and misaligned accesses), racecheck (shared-memory hazards), synccheck
(illegal barrier use) and initcheck (reads of uninitialised device memory) must report 0 errors
on a tiny graph through every kernel family: tcgen05 typed GEMM, narrow / wide / ring walks,
fused tcgen05 backward, tcgen05 dW GEMM (unfused backward), tf32 GEMM + dX source walk, HGT,
and the fp32 layer's 3xTF32 typed and dW GEMMs.
The logs go to gpurun_out/sanitize/ when that directory exists (copied to profiles/ per round).
"""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck", "initcheck"])
@pytest.mark.parametrize("variant", ["fused", "unfused", "f32"])
def test_sanitizer_clean(tool, variant):
    if not os.path.exists(SAN):
        pytest.skip("compute-sanitizer not found")
    cmd = [SAN, "--tool", tool, "--error-exitcode", "9", "--print-limit", "50"]
    if tool == "memcheck":
        cmd += ["--leak-check", "no"]
    if tool == "racecheck":
        cmd += ["--racecheck-report", "all"]
    # racecheck instruments every shared-memory access (minutes per kernel): the RGAT d = 64 path
    # (tcgen05 GEMM, walks, fused / unfused backward with their mbarrier rings, tf32 GEMM + dX walks)
    cmd += [sys.executable, os.path.join(ROOT, "tools", "sanitize_case.py"), variant,
            "rgat64" if tool == "racecheck" else "full"]
    # no caching allocator (memcheck sees every tensor's bounds); the pipelines' 10 s deadlock
    # watchdog is lifted (the tools slow the kernels down by orders of magnitude)
    env = dict(os.environ, PYTORCH_NO_CUDA_MEMORY_CACHING="1", RGNN_WATCHDOG_S="100000")
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1500, env=env, cwd=ROOT)
    log = r.stdout + r.stderr
    out = os.path.join(ROOT, "gpurun_out", "sanitize")
    if os.path.isdir(os.path.join(ROOT, "gpurun_out")):
        os.makedirs(out, exist_ok=True)
        with open(os.path.join(out, f"{tool}_{variant}.log"), "w") as f:
            f.write(" ".join(cmd) + "\n" + log)
    if "is closed on this pool" in log:
        # the GPU pool's compute-sanitizer wrapper refuses to run (a pool policy, not a result);
        # the clean logs of the runs made while it was open are in profiles/r02/sanitize/
        pytest.skip("compute-sanitizer disabled on this GPU pool")
    assert "sanitize case ok" in log, log[-3000:]
    if tool == "racecheck":
        unknown = [h for h in _hazards(log) if not _stage_refill(h)]
        assert not unknown, "\n\n".join(unknown[:5])
        return
    assert "ERROR SUMMARY: 0 errors" in log, log[-3000:]
    assert r.returncode == 0, log[-3000:]


def _hazards(log):
    """The racecheck reports (one string per 'Potential ... hazard' block)."""
    blocks, cur = [], None
    for line in log.splitlines():
        if "hazard detected" in line:
            if cur:
                blocks.append("\n".join(cur))
            cur = [line]
        elif cur is not None and ("Thread" in line or "Value" in line):
            cur.append(line)
    if cur:
        blocks.append("\n".join(cur))
    return blocks


def _stage_refill(h):
    """The one report racecheck cannot order: in k_bwd_fused_tc a compute thread writes its dZ line into
    stage slot s (generic proxy), its warp fences (fence.proxy.async), __syncwarp()s and lane 0 arrives
    on b_full[s]; the MMA thread waits on b_full[s], issues the MMAs that read the slot, commits them
    to empty[s] and also arrives on empty[s] itself; a producer thread waits on empty[s] before its
    cp.async refills the slot.  That chain orders the two writes, but racecheck does not treat a
    warp-aggregated arrive (lane 0 after __syncwarp) as a release for the other lanes, so it reports
    the refill as a WAW / WAR hazard.  Only that exact pair (a k_bwd_fused_tc write or read against a
    cp_async16 refill) is accepted here; any other report fails the test."""
    return "k_bwd_fused_tc" in h and "cp_async16" in h and h.count("Thread") == 2
