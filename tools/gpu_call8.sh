mkdir -p gpurun_out/c8
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py tests/test_gpu_compact.py tests/test_gpu_dx.py tests/test_gpu_hgt.py -x -q > gpurun_out/c8/pytest_g3.log 2>&1; echo "rc $?" >> gpurun_out/c8/pytest_g3.log
for c in am wikikg2 mutag bgs; do timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(\"$c\", round(d[\"ms_per_step\"],3), d[\"phases_ms_per_step\"])" >> gpurun_out/c8/g3.txt; done
