mkdir -p gpurun_out/c4
mv variants/trace.so /tmp/trace.so
cp paper_2301_06284_b200/librgnn.so /tmp/base.so; cp /tmp/trace.so paper_2301_06284_b200/librgnn.so
bash tools/gpu_call3.sh; cp /tmp/base.so paper_2301_06284_b200/librgnn.so
