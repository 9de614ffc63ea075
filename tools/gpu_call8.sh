mkdir -p gpurun_out/c8
timeout 1200 bash tools/variants.sh am mag > gpurun_out/c8/variants_usm.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_compact.py tests/test_gpu_bwd_tm.py -x -q > gpurun_out/c8/pytest_usm.log 2>&1; echo "rc $?" >> gpurun_out/c8/pytest_usm.log
