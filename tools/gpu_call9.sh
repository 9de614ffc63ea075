mkdir -p gpurun_out/c9
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/c9/pytest.log 2>&1; echo "rc $?" >> gpurun_out/c9/pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c9/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/c9/bench_default.json 2> gpurun_out/c9/bench_default.err
