#!/usr/bin/env python
"""bench.py -- one RGAT / RGCN layer forward + backward step on B200.

Default workload: BASELINE.json configs[3], the ogbn-mag-shaped heterograph
(1.94M nodes, 21.1M edges, 4 relations), RGAT, d_in = d_out = 128, bf16
operands (tcgen05 typed GEMM path), dst-partitioned over the ranks.  A step
is one full pass of the hot path: RGAT forward (typed GEMM, fused score /
edge softmax / aggregate) + backward (backward walk, segmented dW GEMM, dW /
dA), plus -- for N > 1 -- the NCCL gather of Y and all-reduce of dW / dA.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config mag|am|wikikg2|bgs|mutag|aifb]
                  [--impl ours|reference]

Prints ONE JSON line on rank 0.  Inputs are synthetic (synth/, seeded) and
larger than L2 for the default config (X 497 MB, Z 5.4 GB), so no flush is
needed between steps.  `--impl reference` times the fp64 CPU oracle on a
bounded sample of the same workload (rank 0 only; other ranks exit 0).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "RGAT/RGCN layer fwd+bwd edges/sec"
UNIT = "edges/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)   # SURVEY 8(d) protocol: 20 warm-up, >= 100 timed
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--config", default="mag")
    ap.add_argument("--model", default=None, choices=[None, "rgcn", "rgat", "hgt"])
    ap.add_argument("--prec", default=None)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--slope", type=float, default=0.2)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="target oracle time of the cpu_baseline sample")
    ap.add_argument("--eager", action="store_true", help="time eager launches instead of a captured CUDA graph")
    ap.add_argument("--dx", action="store_true", help="also compute the input-feature gradient dX (NEXT-2)")
    ap.add_argument("--aggregate-first", action="store_true",
                    help="RGCN: aggregate-first forward (NEXT-4: run-piece sums of x_src, GEMM over the pieces)")
    ap.add_argument("--comm", default="nccl", choices=["nccl", "peer"],
                    help="N>1: NCCL collectives, or the peer-memory communicator (CUDA IPC; the walk stores Y rows "
                         "into every rank's Y_full itself, device-side barrier)")
    ap.add_argument("--gather-sync", action="store_true", help="N>1: gather Y on the caller's stream (no overlap)")
    ap.add_argument("--gather-bf16", action="store_true", help="N>1: gather Y_full in bf16 (half the volume)")
    ap.add_argument("--comm-variants", action="store_true",
                    help="also time compute-only / synchronous / overlapped / bf16 gathers (always on for N>1; "
                         "at N=1 a one-rank communicator exercises the same path)")
    ap.add_argument("--materialization", default="auto", choices=["vanilla", "compact", "auto"],
                    help="per-edge (vanilla) or per-(etype, src) (compact, PAPER.md P:513-531) Z / s_src rows; "
                         "auto = compact when U < E (RGCN) / U <= 3E/4 (RGAT)")
    return ap.parse_args()


def workload(args):
    cfg = synth.get_config(args.config)
    model = args.model or cfg.model
    prec = args.prec or cfg.prec
    return cfg, model, prec


L2_BYTES = 126 * 1024 * 1024


def working_set_bytes(cfg, prec, g):
    b = 2 if prec == "bf16" else 4
    return g.V * cfg.K * b + 2 * g.E * cfg.N * b + 2 * g.V * cfg.N * 4 + 16 * g.E


def needs_flush(cfg, prec, g):
    return working_set_bytes(cfg, prec, g) < 4 * L2_BYTES


def config_json(cfg, model, prec, g, world):
    ws = working_set_bytes(cfg, prec, g)
    l2 = ("L2 flushed between timed steps (write of a 512 MB buffer outside the per-step events); working set %.0f MB"
          % (ws / 1e6)) if needs_flush(cfg, prec, g) else (
        "no flush: per-step inputs larger than L2 (X %.0f MB, Z %.0f MB)" % (
            g.V * cfg.K * (2 if prec == "bf16" else 4) / 1e6, g.E * cfg.N * (2 if prec == "bf16" else 4) / 1e6))
    return {"workload": f"{cfg.name}-shaped heterograph, {model.upper()} layer "
                        f"fwd+bwd, d={cfg.K}",
            "model": model, "prec": prec, "V": int(g.V), "E": int(g.E), "R": int(g.R), "d_in": cfg.K,
            "d_out": cfg.N, "seeds": "graph 0, X 1, W 2, A 3, dY 4 (synth/)", "l2": l2,
            "parallelism": f"dst-range partition x{world} (NCCL Y gather overlapped with the backward + dW "
                           f"all-reduce)" if world > 1 else "1 GPU"}


# --------------------------------------------------------------------- algorithmic bytes
def algorithmic_bytes(phase, model, prec, K, N, E, V_own, J, num_items, U=None):
    """Bytes the method must move per launch of each phase (no L2 reuse assumed).
    U = compact rows (compact materialisation): the GEMM runs over U rows, the
    walks read Z through a per-slot row index (plus 1/c per slot for RGCN)."""
    b = 2 if prec == "bf16" else 4
    if phase == "gemm_fwd":  # gather X rows, write Z, read src index (+ s_src write for RGAT, + 1/c read for RGCN)
        return (E if U is None else U) * (K * b + N * b + 4 + 4)
    if phase == "aggregate" and model == "hgt":  # per edge: slot row, kw and m rows (fp32); per row q, Y, lse, item
        return E * (4 + 2 * N * 4) + num_items * (N * 4 + N * 4 + 4 + 16)
    if phase == "hgt_bwd_walk":  # per edge: slot pos (+ row), kw and m rows (fp32), alpha/da writes; per row q, G, Y, dq
        return E * (4 + (4 if U is not None else 0) + 2 * N * 4 + 8) + num_items * (4 * N * 4 + 4 + 16)
    if phase == "aggregate":  # read pos, et, Z row (+ s_src) per edge; X_dst, Y, lse, item per row
        per_e = N * b + 8 + (4 if model == "rgat" or U is not None else 0)
        per_v = (K * b + N * 4 + 4 + 16) if model == "rgat" else (N * 4 + 16)
        return E * per_e + num_items * per_v
    if phase == "bwd_traverse":  # read pos, et, s_src, Z; write dZ, dpre; per row X, Y, dY, lse, item
        return E * (2 * N * b + 16) + num_items * (K * b + 2 * N * 4 + 4 + 16)
    if phase == "bwd_fused":
        if model == "rgcn":  # gather X_src, read src, dst, 1/c per edge; G_v per (etype, dst) run
            return E * (K * b + 12) + J * 4 * N
        # read Z, s_src, dst, src (+ compact row) per edge, gather X_src; per run G_v, Y_v, X_v, lse
        return E * (N * b + K * b + 12 + (4 if U is not None else 0)) + J * (8 * N + K * b + 4)
    if phase == "bwd_tm":  # RGAT, messages recomputed (bwd_tm.cu): per edge gather X_src, read src, dst, s_src
        # (+ compact row), write dpre; per (etype, dst) run G_v, Y_v (fp32), x_v, lse
        return E * (K * b + 16 + (4 if U is not None else 0)) + J * (8 * N + K * b + 4)
    if phase == "dst_term":  # read dst, dpre per edge; x_v per run
        return E * 8 + J * K * b
    if phase == "gemm_dw":  # gather X rows, read dZ (RGAT) or gather G rows (RGCN), indices; dst term per run
        if model == "rgat":
            return E * (K * b + N * b + 4 + 4 + 4) + J * K * b
        return E * (K * b + N * 4 + 4 + 4 + 4)
    return 0


def sample_clocks_start(path):
    try:
        return subprocess.Popen(
            ["nvidia-smi", "--query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
             "--format=csv,noheader,nounits", "-lms", "200"], stdout=open(path, "w"), stderr=subprocess.DEVNULL)
    except Exception:
        return None


def sample_clocks_stop(proc, path, gpu_index):
    if proc is None:
        return None
    proc.terminate()
    try:
        proc.wait(timeout=5)
    except Exception:
        proc.kill()
    sm, mx, reasons = [], 0.0, set()
    names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
    try:
        for line in open(path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9 or not f[0].isdigit() or int(f[0]) != gpu_index:
                continue
            try:
                sm.append(float(f[1])); mx = max(mx, float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
    except FileNotFoundError:
        return None
    if not sm:
        return None
    load = [x for x in sm if x > 0.5 * mx] or sm
    return {"sm_mhz": float(np.median(load)), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return float(d["hbm_gbs"]), float(d["bf16_tflops"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, 1590.0, "fallback (B200_PROFILING.md)"


# --------------------------------------------------------------------- oracle (cpu baseline / reference arm)
def oracle_sample(g, t, model, K, N, target_s, slope, prec):
    """Contiguous dst range [a, b) of the same graph sized for ~target_s of oracle fwd+bwd."""
    import oracle
    tt = t
    if prec == "bf16":
        sys.path.insert(0, os.path.join(ROOT, "tests"))
        from parity import bf16_inputs
        tt = bf16_inputs(t)
    X, W, A = (np.ascontiguousarray(a, dtype=np.float64) for a in (tt.X, tt.W, tt.A))
    hw = None
    if model == "hgt":
        h = synth.make_hgt_tensors(g.V, g.R, g.T, K, N)
        if prec == "bf16":
            from parity import bf16_round
            hw = [bf16_round(a).astype(np.float64) for a in (h.WK, h.WQ, h.WV, h.Wa, h.Wm)]
        else:
            hw = [a.astype(np.float64) for a in (h.WK, h.WQ, h.WV, h.Wa, h.Wm)]
    W0 = np.ascontiguousarray(tt.W0, dtype=np.float64)
    indeg = np.r_[0, np.cumsum(np.bincount(g.dst, minlength=g.V))]
    a = g.V // 3
    G = np.zeros((g.V, N))

    def run(ne):
        b = int(min(g.V, np.searchsorted(indeg, indeg[a] + ne)))
        b = max(b, a + 1)
        G[a:b] = t.dY[a:b]
        t0 = time.perf_counter()
        if model == "hgt":
            oracle.hgt_forward(g.V, g.R, g.src, g.dst, g.etype, g.ntype, X, *hw, rows=np.arange(a, b))
            oracle.hgt_backward(g.V, g.R, g.src, g.dst, g.etype, g.ntype, X, *hw, G, v0=a, v1=b)
        elif model == "rgat":
            oracle.rgat_forward(g.V, g.R, g.src, g.dst, g.etype, X, W, A, slope=slope, rows=np.arange(a, b))
            oracle.rgat_backward(g.V, g.R, g.src, g.dst, g.etype, X, W, A, G, slope=slope, v0=a, v1=b)
        else:
            oracle.rgcn_forward(g.V, g.R, g.src, g.dst, g.etype, X, W, None, rows=np.arange(a, b))
            oracle.rgcn_backward(g.V, g.R, g.src, g.dst, g.etype, X, G, K, N, v0=a, v1=b)
        dt = time.perf_counter() - t0
        G[a:b] = 0
        return int(indeg[b] - indeg[a]), dt, (a, b)

    # two-point fit t(n) = a + b n (a = the O(E) in-list build and fixed costs)
    n1, t1, _ = run(2000)
    n2, t2, _ = run(40000)
    slope_t = max((t2 - t1) / max(n2 - n1, 1), 1e-9)
    fixed_t = max(t1 - slope_t * n1, 0.0)
    want = int(max(2000, min(g.E, (target_s - fixed_t) / slope_t)))
    return run, want, oracle.num_threads()


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg, model, prec = workload(args)
    g = synth.make_graph(cfg)
    t = synth.make_tensors(g.V, g.R, cfg.K, cfg.N)
    per_step = max(1.0, min(10.0, 150.0 / max(1, args.steps + args.warmup)))
    run, want, cores = oracle_sample(g, t, model, cfg.K, cfg.N, per_step, args.slope, prec)
    for _ in range(args.warmup):
        run(want)
    tot_e, tot_s, rng = 0, 0.0, None
    for _ in range(args.steps):
        ne, dt, rng = run(want)
        tot_e += ne
        tot_s += dt
    v = tot_e / tot_s
    sample = (f"dst rows [{rng[0]},{rng[1]}) of the {cfg.name}-shaped graph ({tot_e // max(args.steps, 1)} in-edges, "
              f"{model} fwd+bwd in fp64), per step")
    out = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": 1e3 * tot_s / args.steps, "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": config_json(cfg, model, prec, g, 1),
           "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
           "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


# --------------------------------------------------------------------- our arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2301_06284_b200 as m

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    cfg, model, prec = workload(args)
    K, N = cfg.K, cfg.N
    t_gen = time.perf_counter()
    g = synth.make_graph(cfg)
    t = synth.make_tensors(g.V, g.R, K, N)
    t_gen = time.perf_counter() - t_gen
    indeg = np.r_[0, np.cumsum(np.bincount(g.dst, minlength=g.V))]
    bounds = m.partition_dst(indeg, world)
    v0, v1 = int(bounds[rank]), int(bounds[rank + 1])

    # preprocessing (timed separately, not part of the step).  A tiny graph is created first so the
    # library's lazily loaded kernels (CUDA module loading) are not charged to the timed creation.
    tiny = synth.random_graph(64, 256, g.R, seed=1)
    m.Graph(tiny.V, tiny.src, tiny.dst, tiny.etype, tiny.R, materialization=args.materialization,
            build_dx=args.dx or model == "hgt", ntype=tiny.ntype if model == "hgt" else None,
            num_ntypes=1 if model == "hgt" else 0, device=dev)
    src = torch.from_numpy(g.src).to(dev); dst = torch.from_numpy(g.dst).to(dev)
    et = torch.from_numpy(g.etype).to(dev)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    G = m.Graph(g.V, src, dst, et, g.R, dst_begin=v0, dst_end=v1, materialization=args.materialization,
                build_dx=args.dx or model == "hgt", ntype=g.ntype if model == "hgt" else None,
                num_ntypes=g.T if model == "hgt" else 0, aggregate_first=args.aggregate_first, device=dev)
    torch.cuda.synchronize()
    prep_ms = 1e3 * (time.perf_counter() - t0)
    del src, dst, et

    xdt = torch.bfloat16 if prec == "bf16" else torch.float32
    X = torch.from_numpy(t.X).to(dev).to(xdt)
    W = torch.from_numpy(t.W).to(dev)
    A = torch.from_numpy(t.A).to(dev)
    dY = torch.from_numpy(np.ascontiguousarray(t.dY[v0:v1])).to(dev)
    ws = m.Workspace(G, model, K, N, prec, dx=args.dx)
    dX = torch.empty(g.V, K, dtype=torch.float32, device=dev) if args.dx else None
    use_comm = world > 1 or args.comm_variants
    # multi-GPU default: the Y gather is asynchronous (overlapped with the backward, which reads only
    # the owned rows) and joined at the end of the step; --gather-sync / --gather-bf16 for A/B
    gather_bf16 = args.gather_bf16
    Y_full = (torch.empty(g.V, N, dtype=torch.bfloat16 if gather_bf16 else torch.float32, device=dev)
              if use_comm else None)
    Y = (Y_full[v0:v1] if use_comm and not gather_bf16
         else torch.empty(v1 - v0, N, dtype=torch.float32, device=dev))
    dW = torch.empty(g.R, K, N, dtype=torch.float32, device=dev)
    dA = torch.empty(g.R, 2, N, dtype=torch.float32, device=dev) if model == "rgat" else None
    comm = None
    if use_comm and args.comm == "peer":
        if gather_bf16:
            raise SystemExit("--gather-bf16 does not apply to --comm peer (fp32 Y_full)")
        comm = m.PeerComm(bounds, rank, world, Y_full, g.R * K * N + g.R * 2 * N + K * N)
    elif use_comm:
        comm = m.Comm(bounds, rank, world)
        comm.set_options(gather_async=not args.gather_sync, gather_bf16=gather_bf16)
    stream = torch.cuda.current_stream(dev)

    HW = None
    hgrads = None
    if model == "hgt":
        h = synth.make_hgt_tensors(g.V, g.R, g.T, K, N)
        HW = [torch.from_numpy(a).to(dev) for a in (h.WK, h.WQ, h.WV, h.Wa, h.Wm)]
        dY = torch.from_numpy(np.ascontiguousarray(h.dY[v0:v1])).to(dev)

    def fwd(Xs=X, Ws=W, As=A, HWs=None):
        if model == "hgt":
            m.hgt_forward(G, Xs, *(HWs or HW), prec=prec, ws=ws, Y=Y, comm=comm, Y_full=Y_full)
        elif model == "rgat":
            m.rgat_forward(G, Xs, Ws, As, args.slope, prec=prec, ws=ws, Y=Y, comm=comm, Y_full=Y_full)
        else:
            m.rgcn_forward(G, Xs, Ws, prec=prec, ws=ws, Y=Y, comm=comm, Y_full=Y_full)

    def bwd(Xs=X, Ws=W, As=A, dYs=dY, HWs=None):
        nonlocal hgrads
        if model == "hgt":  # dWK, dWQ, dWV, dWa, dWm
            hgrads = m.hgt_backward(G, Xs, *(HWs or HW), Y, dYs, ws, prec=prec, comm=comm)
            return
        m.rgnn_backward(G, model, Xs, Ws, dYs, ws, A=As if model == "rgat" else None, slope=args.slope, Y=Y,
                        prec=prec, comm=comm, dW=dW, dA=dA, want_dx=args.dx, dX=dX)

    def step(Xs=X, Ws=W, As=A, dYs=dY, HWs=None):
        fwd(Xs, Ws, As, HWs)
        bwd(Xs, Ws, As, dYs, HWs)
        if comm is not None:
            comm.join()  # Y_full complete before the step ends

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step()
    barrier()
    # The timed step is a captured CUDA graph of the same library calls (the library is
    # capture-safe: caller-owned buffers, stream-ordered launches); --eager times launches.
    use_graph = not args.eager
    graph = None
    if use_graph:
        cap_stream = torch.cuda.Stream(dev)
        cap_stream.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(cap_stream):
            step()  # warm the capture stream
            torch.cuda.synchronize()
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=cap_stream):
                step()
        torch.cuda.synchronize()
        graph.replay()
        barrier()
    run_step = graph.replay if use_graph else step
    clk_path = os.path.join("/tmp", f"rgnn_clocks_{os.getpid()}.csv")
    clk = sample_clocks_start(clk_path) if local == 0 or world == 1 else None
    time.sleep(0.3 if clk else 0)
    flush = needs_flush(cfg, prec, g)
    fbuf = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device=dev) if flush else None
    l0 = m.launch_count()
    if not flush:  # inputs larger than L2: one event pair around the K steps
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        e0.record(stream)
        for _ in range(args.steps):
            run_step()
        e1.record(stream)
        barrier()
        ms = e0.elapsed_time(e1) / args.steps
    else:  # small working set: flush L2 between steps, time each step with its own events
        evs = []
        barrier()
        for _ in range(args.steps):
            fbuf.fill_(1)
            a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a_.record(stream)
            run_step()
            b_.record(stream)
            evs.append((a_, b_))
        barrier()
        ms = sum(a_.elapsed_time(b_) for a_, b_ in evs) / args.steps
    clocks = sample_clocks_stop(clk, clk_path, local)
    if use_graph:  # kernels launched per step, counted on one eager step
        l1 = m.launch_count()
        step()
        torch.cuda.synchronize()
        launches = (m.launch_count() - l1) * args.steps
    else:
        launches = m.launch_count() - l0
    # per-phase device time (live CUDA events on the launching stream) from an eager pass
    m._binding.profile_enable(True)
    m._binding.profile_read()
    barrier()
    for _ in range(args.steps):
        if flush:
            fbuf.fill_(1)
        step()
    barrier()
    phases = m._binding.profile_read()
    m._binding.profile_enable(False)
    # per-step distribution: fwd, bwd and fwd+bwd of each eager step by CUDA events
    ev = []
    barrier()
    for _ in range(args.steps):
        if flush:
            fbuf.fill_(1)
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record(stream)
        fwd()
        e[1].record(stream)
        bwd()
        e[2].record(stream)
        ev.append(e)
    barrier()

    def pct(xs):
        return {"p10": round(float(np.percentile(xs, 10)), 4), "p50": round(float(np.percentile(xs, 50)), 4),
                "p90": round(float(np.percentile(xs, 90)), 4)}
    step_pct = {"fwd": pct([e[0].elapsed_time(e[1]) for e in ev]), "bwd": pct([e[1].elapsed_time(e[2]) for e in ev]),
                "fwd+bwd": pct([e[0].elapsed_time(e[2]) for e in ev]), "launch": "eager", "steps": len(ev)}
    if world > 1:  # max over ranks
        tm = torch.tensor([ms], device=dev)
        dist.all_reduce(tm, op=dist.ReduceOp.MAX)
        ms = float(tm.item())
    value = g.E / (ms * 1e-3)

    # ---- multi-GPU reporting: compute-only (sharded Y, no gather) and the step with a
    # synchronous, an overlapped (asynchronous, joined at step end) and a bf16 overlapped gather;
    # eager steps timed by CUDA events, max over ranks
    multi = None
    if comm is not None:
        def timed_events(fn, n):
            fn()
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(n):
                fn()
            e1.record(stream)
            barrier()
            t_ = torch.tensor([e0.elapsed_time(e1) / n], device=dev)
            if world > 1:
                dist.all_reduce(t_, op=dist.ReduceOp.MAX)
            return float(t_.item())

        nvar = max(3, min(args.steps, 10))
        saved_full = Y_full

        def variant(flags_async, flags_bf16, with_gather=True):
            nonlocal Y_full
            comm.set_options(gather_async=flags_async, gather_bf16=flags_bf16)
            if not with_gather:
                Y_full = None
            elif flags_bf16 != gather_bf16:
                Y_full = torch.empty(g.V, N, dtype=torch.bfloat16 if flags_bf16 else torch.float32, device=dev)
            else:
                Y_full = saved_full
            try:
                return timed_events(step, nvar)
            finally:
                Y_full = saved_full
                comm.set_options(gather_async=not args.gather_sync, gather_bf16=gather_bf16)

        yb = (g.V * N * 4, g.V * N * 2)
        if args.comm == "peer":
            multi = {"compute_only_ms": variant(False, False, with_gather=False),
                     "peer_fused_gather_ms": variant(False, False),
                     "y_gather_bytes_per_rank": {"fp32": int(yb[0] * (world - 1) / max(world, 1))},
                     "steps": nvar, "launch": "eager", "default": "peer-memory (walk epilogue stores + barrier)"}
    if comm is not None and args.comm != "peer":
        multi = {"compute_only_ms": variant(True, gather_bf16, with_gather=False),
                 "gather_sync_ms": variant(False, False), "gather_overlapped_ms": variant(True, False),
                 "gather_overlapped_bf16_ms": variant(True, True),
                 "y_gather_bytes_per_rank": {"fp32": int(yb[0] * (world - 1) / max(world, 1)),
                                             "bf16": int(yb[1] * (world - 1) / max(world, 1))},
                 "steps": nvar, "launch": "eager", "default": "overlapped" + (" bf16" if gather_bf16 else "")
                 if not args.gather_sync else "sync"}

    # ---- end to end through the public API with host buffers (pinned), copies inside the timed region
    e2e = None
    if not args.no_e2e:
        hX = t.X.astype(np.float32)
        hX = torch.from_numpy(hX).to(xdt).pin_memory()
        hW = torch.from_numpy(t.W).pin_memory(); hA = torch.from_numpy(t.A).pin_memory()
        hdY = torch.from_numpy(np.ascontiguousarray(t.dY[v0:v1])).pin_memory()
        oY = torch.empty(v1 - v0, N, dtype=torch.float32).pin_memory()
        odW = torch.empty(g.R, K, N, dtype=torch.float32).pin_memory()
        odA = torch.empty(g.R, 2, N, dtype=torch.float32).pin_memory() if dA is not None else None
        dX_, dW_, dA_, ddY = torch.empty_like(X), torch.empty_like(W), torch.empty_like(A), torch.empty_like(dY)
        h2d = hX.numel() * hX.element_size() + hW.numel() * 4 + hA.numel() * 4 + hdY.numel() * 4
        odX = torch.empty(g.V, K, dtype=torch.float32).pin_memory() if args.dx else None
        d2h = oY.numel() * 4 + odW.numel() * 4 + (odA.numel() * 4 if odA is not None else 0) + (
            odX.numel() * 4 if odX is not None else 0)
        n_e2e = max(1, min(args.steps, 5))

        if model == "hgt":
            hHW = [a.cpu().pin_memory() for a in HW]
            dHW = [torch.empty_like(a) for a in HW]
            hdY = dY.cpu().pin_memory()
            ohg = [torch.empty(a.shape, dtype=torch.float32).pin_memory() for a in HW]
            h2d = hX.numel() * hX.element_size() + sum(a.numel() * 4 for a in hHW) + hdY.numel() * 4
            d2h = oY.numel() * 4 + sum(a.numel() * 4 for a in ohg)

        s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)

        def e2e_step():
            # X and the weights are copied in first; dY streams in on a side stream while the forward
            # runs (it is needed only by the backward) and Y streams out while the backward runs
            # (PCIe is full duplex); gradients are copied out after the backward.
            main = torch.cuda.current_stream(dev)
            dX_.copy_(hX, non_blocking=True)
            if model == "hgt":
                for a, b in zip(dHW, hHW):
                    a.copy_(b, non_blocking=True)
            else:
                dW_.copy_(hW, non_blocking=True)
                dA_.copy_(hA, non_blocking=True)
            s_in.wait_stream(main)
            with torch.cuda.stream(s_in):
                ddY.copy_(hdY, non_blocking=True)
            fwd(dX_, dW_, dA_, HWs=dHW if model == "hgt" else None)
            s_out.wait_stream(main)
            with torch.cuda.stream(s_out):
                oY.copy_(Y, non_blocking=True)
            main.wait_stream(s_in)
            bwd(dX_, dW_, dA_, ddY, HWs=dHW if model == "hgt" else None)
            if model == "hgt":
                for o, gr in zip(ohg, hgrads):
                    o.copy_(gr, non_blocking=True)
            else:
                odW.copy_(dW, non_blocking=True)
                if odA is not None:
                    odA.copy_(dA, non_blocking=True)
                if odX is not None:
                    odX.copy_(dX, non_blocking=True)
            main.synchronize()  # the host reads the results every step
            s_out.synchronize()

        def timed(fn):
            fn()
            barrier()
            t0 = time.perf_counter()
            for _ in range(n_e2e):
                fn()
            barrier()
            ems = 1e3 * (time.perf_counter() - t0) / n_e2e
            if world > 1:
                tm = torch.tensor([ems], device=dev)
                dist.all_reduce(tm, op=dist.ReduceOp.MAX)
                ems = float(tm.item())
            return ems

        ems = timed(e2e_step)
        e2e_io = {"value": g.E / (ems * 1e-3), "unit": UNIT, "ms_per_step": ems, "h2d_bytes_per_step": int(h2d),
                  "d2h_bytes_per_step": int(d2h), "steps": n_e2e,
                  "protocol": "layer I/O: X, W (A) and dY in, Y and the gradients out every step",
                  "pipelining": "X, W in then forward; dY copied in on a side stream during the forward, Y copied "
                                "out on a side stream during the backward; gradients out after it"}

        # Training step of the paper's protocol (NLL loss on random labels): X, the weights and
        # the labels in; forward; loss = NLL(log_softmax(Y)) and dY = d loss / dY on the device (torch,
        # the caller's loss -- not part of the layer); backward; the loss and the gradients out.
        lab = np.random.Generator(np.random.PCG64(5)).integers(0, N, size=g.V)  # label_seed = 5
        hlab = torch.from_numpy(np.ascontiguousarray(lab[v0:v1])).pin_memory()
        dlab = torch.empty_like(hlab, device=dev)
        oloss = torch.empty(1, dtype=torch.float32).pin_memory()
        nll_scale = 1.0 / g.V  # mean over all V rows (every rank owns a slice)

        # All of a step's inputs (X, the weights, the labels) are double-buffered: step i+1's inputs are
        # copied in on a side stream while step i runs (one upload per timed step, inside the timed
        # region).  The small copies go first and the whole set is awaited with one event, so no
        # small per-step copy queues behind the 0.5 GB X copy on the host-to-device engine.
        s_up = torch.cuda.Stream(dev)
        ev_up = [torch.cuda.Event(), torch.cuda.Event()]
        ibuf = [{"X": dX_, "W": dW_, "A": dA_, "lab": dlab, "HW": dHW if model == "hgt" else None},
                {"X": torch.empty_like(dX_), "W": torch.empty_like(dW_), "A": torch.empty_like(dA_),
                 "lab": torch.empty_like(dlab),
                 "HW": [torch.empty_like(a) for a in dHW] if model == "hgt" else None}]
        tstate = {"i": 0}

        def upload(b):
            with torch.cuda.stream(s_up):
                b["lab"].copy_(hlab, non_blocking=True)
                if model == "hgt":
                    for a, h in zip(b["HW"], hHW):
                        a.copy_(h, non_blocking=True)
                else:
                    b["W"].copy_(hW, non_blocking=True)
                    b["A"].copy_(hA, non_blocking=True)
                b["X"].copy_(hX, non_blocking=True)

        upload(ibuf[0])
        ev_up[0].record(s_up)

        def train_step():
            main = torch.cuda.current_stream(dev)
            i = tstate["i"]
            cb, nb = ibuf[i % 2], ibuf[(i + 1) % 2]
            main.wait_event(ev_up[i % 2])          # this step's inputs have landed
            s_up.wait_stream(main)                 # (the previous step, which read nb, is done)
            upload(nb)                             # next step's inputs under this step's compute
            ev_up[(i + 1) % 2].record(s_up)
            tstate["i"] = i + 1
            cur, dW_c, dA_c, dlab_c, dHW_c = cb["X"], cb["W"], cb["A"], cb["lab"], cb["HW"]
            fwd(cur, dW_c, dA_c, HWs=dHW_c)
            lp = torch.log_softmax(Y, dim=1)
            loss = -lp.gather(1, dlab_c.view(-1, 1)).sum() * nll_scale
            dyy = lp.exp_()
            dyy[torch.arange(dyy.shape[0], device=dev), dlab_c] -= 1.0
            dyy.mul_(nll_scale)
            bwd(cur, dW_c, dA_c, dyy, HWs=dHW_c)
            oloss.copy_(loss.view(1), non_blocking=True)
            if model == "hgt":
                for o, gr in zip(ohg, hgrads):
                    o.copy_(gr, non_blocking=True)
            else:
                odW.copy_(dW, non_blocking=True)
                if odA is not None:
                    odA.copy_(dA, non_blocking=True)
            main.synchronize()

        tms = timed(train_step)
        h2d_t = hX.numel() * hX.element_size() + hlab.numel() * 8 + (
            sum(a.numel() * 4 for a in hHW) if model == "hgt" else hW.numel() * 4 + hA.numel() * 4)
        d2h_t = 4 + (sum(a.numel() * 4 for a in ohg) if model == "hgt" else
                     odW.numel() * 4 + (odA.numel() * 4 if odA is not None else 0))
        e2e = {"value": g.E / (tms * 1e-3), "unit": UNIT, "ms_per_step": tms, "h2d_bytes_per_step": int(h2d_t),
               "d2h_bytes_per_step": int(d2h_t), "steps": n_e2e,
               "protocol": "training step (P:843): X, weights and random labels in; forward; NLL(log_softmax(Y)) "
                           "loss and dY on the device (torch, the caller's loss); backward; loss and weight "
                           "gradients out; inputs double-buffered (step i+1's X, weights and labels are copied in "
                           "on a side stream during step i, one upload per timed step)"
                           + ("; dX not computed" if not args.dx else "; dX computed, not copied out"),
               "layer_io": e2e_io}

    # ---- roofline of the dominant kernel phase (live CUDA-event durations from the timed region)
    hbm, tflops, peak_src = peaks()
    v = G.view
    step_phase = {k: (tot / args.steps, n // max(args.steps, 1)) for k, (tot, n) in phases.items()}
    cand = {k: x for k, x in step_phase.items()
            if k in ("gemm_fwd", "aggregate", "bwd_traverse", "gemm_dw", "bwd_fused", "bwd_tm", "hgt_bwd_walk")}
    roof = None
    if cand:
        dom = max(cand, key=lambda k: cand[k][0])
        per_launch_ms = phases[dom][0] / max(phases[dom][1], 1)
        zr = G.zrows(model)
        byts = algorithmic_bytes(dom, model, prec, K, N, int(v.E_own), int(v.V_own), int(v.num_runs),
                                 int(v.num_items), U=zr if zr != int(v.E_own) else None)
        ach = byts / (per_launch_ms * 1e-3) / 1e9
        traffic = None
        try:
            tj = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
            mat = "compact" if zr != int(v.E_own) else "vanilla"
            traffic = tj.get(f"{cfg.name}:{model}:{prec}:{mat}:{dom}")
        except Exception:
            pass
        # compact-minimal bytes (the fused RGAT backward on compact rows: x_src per edge, each unique Z
        # row once, the per-run rows) and the DRAM fraction of the ncu traffic -- the two other views of
        # the same launch
        b_ = 2 if prec == "bf16" else 4
        minimal = byts
        if dom == "bwd_fused" and model == "rgat" and zr != int(v.E_own):
            minimal = int(v.E_own) * (K * b_ + 16) + zr * N * b_ + int(v.num_runs) * (8 * N + K * b_ + 4)
        roof = {"kernel": dom, "bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
                "traffic": traffic, "algorithmic_bytes_per_launch": int(byts), "launch_ms": per_launch_ms,
                "peak_source": peak_src, "minimal_bytes_per_launch": int(minimal),
                "minimal_frac": minimal / (per_launch_ms * 1e-3) / 1e9 / hbm,
                "dram_frac": (traffic / (per_launch_ms * 1e-3) / 1e9 / hbm) if traffic else None}

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:  # rank 0 only (the other ranks wait at the final barrier)
        run, want, cores = oracle_sample(g, t, model, K, N, args.cpu_seconds, args.slope, prec)
        ne, dt, rng = run(want)
        cpu = {"value": ne / dt, "unit": UNIT, "cores": cores, "kind": "oracle",
               "sample": f"dst rows [{rng[0]},{rng[1]}) ({ne} in-edges) of the same graph, {model} fwd+bwd fp64, "
                         f"{dt:.1f} s"}

    if rank == 0:
        out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
               "vs_baseline": None, "dtype": prec, "data": "synthetic (seeded generator, random-init weights)",
               "config": dict(config_json(cfg, model, prec, g, world),
                              launch="CUDA graph of the step" if use_graph else "eager",
                              backward=("dWK, dWQ, dWV, dWa, dWm" if model == "hgt" else
                                        "dW, dA" + (", dX (NEXT-2)" if args.dx else "") if model == "rgat" else
                                        "dW" + (", dX (NEXT-2)" if args.dx else "")),
                              materialization=("aggregate-first (run pieces)" if args.aggregate_first
                                               and model == "rgcn" else
                                               ("compact" if G.zrows(model) != G.E_own else "vanilla") + (
                                  " (auto)" if args.materialization == "auto" else "")),
                              z_rows=G.zrows(model), compact_rows=int(G.num_compact)),
               "clocks": clocks, "e2e": e2e,
               "gpu_launches": int(launches), "roofline": roof, "cpu_baseline": cpu, "multi_gpu": multi,
               "phases_ms_per_step": {k: round(x[0], 4) for k, x in sorted(step_phase.items())},
               "step_ms_percentiles": step_pct,
               "preprocess_ms": G.create_ms, "preprocess_with_alloc_ms": prep_ms, "generate_s": round(t_gen, 1)}
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
