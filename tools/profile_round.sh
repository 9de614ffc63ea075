#!/bin/bash
# ncu evidence for profiles/ (run under gpurun from the repo root; one GPU).
#   launch lists (cold-cache, serialised per-launch times) and --set full captures of the
#   top kernels, plus the tensor-pipe metrics, for the RGAT (default) and HGT mag workloads.
set -x
OUT=gpurun_out/prof
mkdir -p $OUT
B="python bench.py --steps 2 --warmup 3 --eager --no-e2e --no-cpu-baseline"
TP="sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_tc.sum"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_ --csv --log-file $OUT/launches_rgat.csv $B > $OUT/launches_rgat.log 2>&1
timeout 900 ncu --set full --metrics $TP --clock-control none --import-source on \
  -k regex:'k_gemm_fwd_tc|k_aggregate|k_bwd_fused_tc' -c 3 -o $OUT/rgat_full $B > $OUT/rgat_full.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_ --csv --log-file $OUT/launches_hgt.csv $B --model hgt > $OUT/launches_hgt.log 2>&1
timeout 1200 ncu --set full --metrics $TP --clock-control none \
  -k regex:'k_gemm_fwd_tf32|k_aggregate_hgt|k_hgt_bwd_walk|k_hgt_piece_agg|k_gemm_dw_tc|k_dx_walk' -c 16 -o $OUT/hgt_full $B --model hgt > $OUT/hgt_full.log 2>&1
ls -la $OUT
