mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/g1_smi.txt
for f in variants/lib_*.so; do SCV_LIB=$f timeout 120 python tools/stagebench.py 2047 >> gpurun_out/g1_stage.txt 2>&1; done
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/g1_bench.json 2> gpurun_out/g1_bench.err
