#!/bin/bash
# ncu evidence per config (run under gpurun from the repo root; one GPU):
#   launch list (cold-cache, serialised) + one --set full capture of each top kernel, summarised on
#   the box (the .ncu-rep files stay in /tmp: they exceed what gpurun copies back).
#   usage: tools/profile_configs.sh <tag> <kernel-regex> <config>...   (e.g. r02 'k_aggregate|k_bwd_fused_tc' am mag)
TAG=$1; shift
KRE=$1; shift
OUT=gpurun_out/prof_$TAG
REP=/tmp/prof_$TAG
mkdir -p $OUT $REP
TP="sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_tc.sum"
for c in "$@"; do
  B="python bench.py --config $c --steps 2 --warmup 3 --eager --no-e2e --no-cpu-baseline"
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_ --csv \
    --log-file $OUT/launches_$c.csv $B > $OUT/launches_$c.log 2>&1
  python tools/ncu_summarize.py launches $OUT/launches_$c.csv $OUT/launches_summary_$c.txt "$B"
  timeout 1200 ncu --set full --metrics $TP --clock-control none --import-source on \
    -k regex:"$KRE" -c ${NCAP:-4} -o $REP/full_$c $B > $OUT/full_$c.log 2>&1
  python tools/ncu_summarize.py full $REP/full_$c.ncu-rep $OUT/full_summary_$c.json > /dev/null
  for k in $(ncu -i $REP/full_$c.ncu-rep --page raw --csv --metrics launch__grid_size 2>/dev/null | \
             python -c "import csv,sys; r=list(csv.reader(sys.stdin)); i=r[0].index('Kernel Name'); print(' '.join(sorted({x[i].split('(')[0].split('<')[0].replace('void ','').replace('rgnn::','').strip() for x in r[2:]})))"); do
    python tools/ncu_stalls.py $REP/full_$c.ncu-rep "^$k\$" 30 > $OUT/stalls_${c}_$k.txt 2>&1
    python tools/ncu_srclines.py $REP/full_$c.ncu-rep "^$k\$" 40 > $OUT/srclines_${c}_$k.txt 2>&1
  done
  ncu -i $REP/full_$c.ncu-rep --page details > $OUT/details_$c.txt 2>&1
done
ls -la $OUT
