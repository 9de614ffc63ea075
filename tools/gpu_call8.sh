mkdir -p gpurun_out/c8
timeout 1200 bash tools/variants.sh mag > gpurun_out/c8/variants_dst.txt 2>&1
