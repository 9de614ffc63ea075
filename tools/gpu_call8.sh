mkdir -p gpurun_out/c8
timeout 1200 bash tools/variants.sh mag am wikikg2 > gpurun_out/c8/variants.txt 2>&1
cp variants/EMPTY0.so paper_2301_06284_b200/librgnn.so
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_compact.py -x -q > gpurun_out/c8/pytest_empty0.log 2>&1; echo "rc $?" >> gpurun_out/c8/pytest_empty0.log
