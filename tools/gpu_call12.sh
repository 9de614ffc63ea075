mkdir -p gpurun_out/c12
RGNN_WALK_RING=1 RGNN_WALK_BULK=1 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_compact.py -x -q > gpurun_out/c12/pytest_bulk.log 2>&1; echo "rc $?" >> gpurun_out/c12/pytest_bulk.log
for c in mag am wikikg2; do
 for v in "" "RGNN_WALK_RING=1" "RGNN_WALK_RING=1 RGNN_WALK_BULK=1"; do
  env $v timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(\"$c [$v]\", round(d[\"ms_per_step\"],3), d[\"phases_ms_per_step\"][\"aggregate\"])" >> gpurun_out/c12/bulk.txt
 done
done
