mkdir -p gpurun_out/c8
timeout 1200 bash tools/variants.sh mag mag > gpurun_out/c8/variants_l1pf.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_bwd_tm.py -x -q > gpurun_out/c8/pytest_l1.log 2>&1; echo "rc $?" >> gpurun_out/c8/pytest_l1.log
