mkdir -p gpurun_out/c2
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_compact.py -x -q -k "rgat or RGAT" > gpurun_out/c2/pytest.log 2>&1; echo "rc $?" >> gpurun_out/c2/pytest.log
for c in mag am; do
  timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/c2/bench_$c.json 2> gpurun_out/c2/bench_$c.err
done
TAG=${TAG:-r02k} KRE="k_bwd_rgat_tm" CONFIGS="mag am" bash tools/gpu_prof.sh > /dev/null 2>&1
