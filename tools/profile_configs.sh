#!/bin/bash
# ncu evidence per config (run under gpurun from the repo root; one GPU):
#   launch list (cold-cache, serialised) + one --set full capture of each top kernel.
#   usage: tools/profile_configs.sh <tag> <config>...   (e.g. r02 am wikikg2 mag)
TAG=$1; shift
OUT=gpurun_out/prof_$TAG
mkdir -p $OUT
TP="sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_tc.sum"
for c in "$@"; do
  B="python bench.py --config $c --steps 2 --warmup 3 --eager --no-e2e --no-cpu-baseline"
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_ --csv \
    --log-file $OUT/launches_$c.csv $B > $OUT/launches_$c.log 2>&1
  timeout 1200 ncu --set full --metrics $TP --clock-control none --import-source on \
    -k regex:'k_gemm_fwd_tc|k_aggregate|k_bwd_fused_tc' -c 4 -o $OUT/full_$c $B > $OUT/full_$c.log 2>&1
done
ls -la $OUT
