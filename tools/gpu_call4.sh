mkdir -p gpurun_out/c4
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_compact.py -x -q -k "rgat or RGAT" > gpurun_out/c4/pytest.log 2>&1; echo "rc $?" >> gpurun_out/c4/pytest.log
mv variants/trace.so /tmp/trace.so
for c in mag; do timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(\"$c\", round(d[\"ms_per_step\"],3), d[\"phases_ms_per_step\"])" >> gpurun_out/c4/variants.txt; done
cp paper_2301_06284_b200/librgnn.so /tmp/base.so; cp /tmp/trace.so paper_2301_06284_b200/librgnn.so
bash tools/gpu_call3.sh; cp /tmp/base.so paper_2301_06284_b200/librgnn.so
