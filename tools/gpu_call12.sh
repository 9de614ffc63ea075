mkdir -p gpurun_out/c12
timeout 900 python -m pytest tests/test_gpu_bwd_tm.py tests/test_gpu_parity.py tests/test_gpu_peer.py -x -q > gpurun_out/c12/pytest_tm.log 2>&1; echo "rc $?" >> gpurun_out/c12/pytest_tm.log
for c in mag mag; do timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(\"$c\", round(d[\"ms_per_step\"],3), d[\"phases_ms_per_step\"])" >> gpurun_out/c12/tm.txt; done
