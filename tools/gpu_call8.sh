mkdir -p gpurun_out/c8
timeout 1500 bash tools/variants.sh mag am > gpurun_out/c8/variants_unr.txt 2>&1
