mkdir -p gpurun_out/c5
timeout 600 python -m pytest tests/test_gpu_bwd_tm.py -q -x > gpurun_out/c5/pytest_tm.log 2>&1; echo "rc $?" >> gpurun_out/c5/pytest_tm.log
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/c5/pytest.log 2>&1; echo "rc $?" >> gpurun_out/c5/pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c5/smoke.log 2>&1
for c in mag am wikikg2; do timeout 600 python bench.py --config $c > gpurun_out/c5/bench_$c.json 2> gpurun_out/c5/bench_$c.err; done
