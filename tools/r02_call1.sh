#!/bin/bash
# r02 first GPU pass: full GPU suite, smoke, bench line, reference arm, ncu launch list
O=gpurun_out; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $O/r02a_smi.txt
free -g > $O/r02a_host.txt; nproc >> $O/r02a_host.txt
timeout 2400 python -m pytest tests -m gpu -x -q > $O/r02a_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/r02a_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/r02a_smoke.log 2>&1
timeout 900 python bench.py > $O/r02a_bench.json 2> $O/r02a_bench.err; echo "bench rc=$?" >> $O/r02a_bench.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/r02a_bench_ref.json 2> $O/r02a_bench_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02a_launches.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/r02a_ncu_launch.log 2>&1
tail -3 $O/r02a_pytest_gpu.log; cat $O/r02a_smoke.log | tail -2; cat $O/r02a_bench.json | cut -c1-1500
