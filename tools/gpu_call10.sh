mkdir -p gpurun_out/c10
timeout 600 python -m pytest tests/test_gpu_bwd_tm.py -q -k "tm2" > gpurun_out/c10/pytest.log 2>&1; echo "rc $?" >> gpurun_out/c10/pytest.log
for m in 1 2; do RGNN_BWD_TM=$m timeout 300 python bench.py --config mag --steps 30 --warmup 5 --no-e2e --no-cpu-baseline 2>gpurun_out/c10/bench_$m.err | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(\"mag tm=$m\", round(d[\"ms_per_step\"],3), d[\"phases_ms_per_step\"])" >> gpurun_out/c10/bench.txt; done
