mkdir -p gpurun_out/c6
for c in mag am; do timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/c6/bench_$c.json 2> gpurun_out/c6/bench_$c.err; done
NCAP=6 bash tools/profile_configs.sh r02final "k_gemm_fwd_tc|k_aggregate|k_bwd_fused_tc|k_bwd_rgat_tm|k_dst_term" mag am wikikg2 > /dev/null 2>&1
