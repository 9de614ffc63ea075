mkdir -p gpurun_out/c11
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/bgb tools/bulk_gather_bench.cu && timeout 300 /tmp/bgb > gpurun_out/c11/bulk.txt 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/gb tools/gather_bench.cu && timeout 300 /tmp/gb > gpurun_out/c11/ldg.txt 2>&1
