mkdir -p gpurun_out/c8
timeout 1200 bash tools/variants.sh am wikikg2 > gpurun_out/c8/variants_gemm.txt 2>&1
cp variants/FWDMINB2.so paper_2301_06284_b200/librgnn.so
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py -x -q > gpurun_out/c8/pytest_gemm.log 2>&1; echo "rc $?" >> gpurun_out/c8/pytest_gemm.log
