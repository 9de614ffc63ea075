mkdir -p gpurun_out/c8
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_compact.py tests/test_gpu_fullsize.py -x -q > gpurun_out/c8/pytest_occ.log 2>&1; echo "rc $?" >> gpurun_out/c8/pytest_occ.log
timeout 1500 bash tools/variants.sh mag am wikikg2 > gpurun_out/c8/variants_occ2.txt 2>&1
