#!/bin/bash
# One bench line per graded config (BASELINE.json configs), for BASELINE.md's table, plus the fp32 layer
# at AM / ogbn-mag size, the aggregate-first RGCN (NEXT-4) and HGT.
mkdir -p gpurun_out/bench_all
for c in mag am wikikg2 bgs mutag aifb; do
  timeout 900 python bench.py --config $c > gpurun_out/bench_all/$c.json 2> gpurun_out/bench_all/$c.err
done
for c in am mag; do
  timeout 900 python bench.py --config $c --prec f32 --no-e2e --no-cpu-baseline > gpurun_out/bench_all/${c}_f32.json 2> gpurun_out/bench_all/${c}_f32.err
done
timeout 900 python bench.py --config wikikg2 --aggregate-first --no-e2e --no-cpu-baseline > gpurun_out/bench_all/wikikg2_aggfirst.json 2> gpurun_out/bench_all/wikikg2_aggfirst.err
timeout 900 python bench.py --model hgt > gpurun_out/bench_all/mag_hgt.json 2> gpurun_out/bench_all/mag_hgt.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_all/reference.json 2> gpurun_out/bench_all/reference.err
