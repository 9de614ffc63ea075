mkdir -p gpurun_out/c8
timeout 600 python -m pytest tests/test_gpu_bwd_tm.py -x -q > gpurun_out/c8/pytest_early.log 2>&1; echo "rc $?" >> gpurun_out/c8/pytest_early.log
timeout 1200 bash tools/variants.sh mag mag bgs > gpurun_out/c8/variants_early.txt 2>&1
