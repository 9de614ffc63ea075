#!/bin/bash
# One bench line per graded config (BASELINE.json configs), for BASELINE.md's table.
mkdir -p gpurun_out/bench_all
for c in mag am wikikg2 bgs mutag aifb; do
  timeout 900 python bench.py --config $c > gpurun_out/bench_all/$c.json 2> gpurun_out/bench_all/$c.err
done
timeout 900 python bench.py --model hgt > gpurun_out/bench_all/mag_hgt.json 2> gpurun_out/bench_all/mag_hgt.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_all/reference.json 2> gpurun_out/bench_all/reference.err
