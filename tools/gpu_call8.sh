mkdir -p gpurun_out/c8
timeout 1500 bash tools/variants.sh mag mag mag > gpurun_out/c8/variants_nobar.txt 2>&1
