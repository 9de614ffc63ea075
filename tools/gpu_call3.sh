mkdir -p gpurun_out
timeout 300 python bench.py --config mag --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --eager > gpurun_out/trace_bench.json 2> gpurun_out/trace_bench.err
python tools/tm_trace.py gpurun_out/tm_trace.txt 10 40 > gpurun_out/tm_trace_mag.txt
