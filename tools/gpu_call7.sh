mkdir -p gpurun_out/c7
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/c7/pytest.log 2>&1; echo "rc $?" >> gpurun_out/c7/pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c7/smoke.log 2>&1
timeout 2400 bash tools/bench_all.sh
