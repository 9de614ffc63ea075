mkdir -p gpurun_out/c8
NCAP=6 bash tools/profile_configs.sh r02final3 "k_bwd_rgat_tm|k_dst_term|k_aggregate" mag > /dev/null 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/c8/pytest_final.log 2>&1; echo "rc $?" >> gpurun_out/c8/pytest_final.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c8/smoke_final.log 2>&1
timeout 600 python bench.py > gpurun_out/c8/bench_final.json 2> gpurun_out/c8/bench_final.err
