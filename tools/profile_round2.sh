#!/bin/bash
# GPU-box pass for one build: default bench line (+real path), ncu launch list
# of the bench command, and --set full captures of the four L=1024 kernels on a
# 16-row beta slab (tools/prof_slab.py).  usage: tools/profile_round2.sh TAG
TAG=${1:-r01}
O=gpurun_out
mkdir -p $O
python bench.py --steps 3 --warmup 3 > $O/bench_$TAG.log 2>&1 || { echo "bench failed"; tail -20 $O/bench_$TAG.log; exit 1; }
tail -1 $O/bench_$TAG.log > $O/bench_$TAG.json
python bench.py --steps 2 --warmup 3 --real --no-cpu-baseline > $O/bench_real_$TAG.log 2>&1; tail -1 $O/bench_real_$TAG.log > $O/bench_real_$TAG.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$TAG.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_launch_$TAG.log 2>&1
for k in k_ana_colgen_s k_pfa_rows k_syn_alpha k_syn_gamma_q; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 -o $O/full_${k}_$TAG \
    python tools/prof_slab.py 1024 16 > $O/ncu_${k}_$TAG.log 2>&1
done
echo done
