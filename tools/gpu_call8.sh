mkdir -p gpurun_out/c8
timeout 600 python -m pytest tests/test_gpu_bwd_tm.py -x -q > gpurun_out/c8/pytest_cw.log 2>&1; echo "rc $?" >> gpurun_out/c8/pytest_cw.log
cp paper_2301_06284_b200/librgnn.so /tmp/b.so; cp variants/CW8.so paper_2301_06284_b200/librgnn.so
timeout 600 python -m pytest tests/test_gpu_bwd_tm.py -x -q > gpurun_out/c8/pytest_cw8.log 2>&1; echo "rc $?" >> gpurun_out/c8/pytest_cw8.log
cp /tmp/b.so paper_2301_06284_b200/librgnn.so
timeout 1500 bash tools/variants.sh mag mag bgs > gpurun_out/c8/variants_cw.txt 2>&1
