mkdir -p gpurun_out/c8
timeout 600 python -m pytest tests/test_gpu_bwd_tm.py -x -q > gpurun_out/c8/pytest_pw.log 2>&1; echo "rc $?" >> gpurun_out/c8/pytest_pw.log
timeout 1500 bash tools/variants.sh mag mag mag > gpurun_out/c8/variants_pw.txt 2>&1
