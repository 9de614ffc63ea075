mkdir -p gpurun_out/c8
timeout 1200 bash tools/variants.sh am wikikg2 > gpurun_out/c8/variants_bwd.txt 2>&1
