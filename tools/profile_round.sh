#!/bin/bash
# GPU-box profiling pass for one round: bench line, ncu launch list (L=1024),
# and one `ncu --set full` capture per top kernel at L=512 (full-size launches
# replay tens of GB of in-place state).  usage: tools/profile_round.sh TAG
TAG=${1:-r01}
O=gpurun_out
mkdir -p $O
python bench.py --steps 2 --warmup 3 > $O/bench_$TAG.log 2>&1 || { echo "bench failed"; tail -20 $O/bench_$TAG.log; exit 1; }
tail -1 $O/bench_$TAG.log > $O/bench_$TAG.json
python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_plain_$TAG.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$TAG.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_launch_$TAG.log 2>&1
python bench.py --L 512 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench512_$TAG.log 2>&1 || exit 1
for k in "k_beta2<.int.11>" "k_ana_gamma<.int.1023>" "k_ana_alpha<.int.1023>" "k_syn_alpha<.int.1023>" "k_syn_gamma<.int.1023>"; do
  n=${k%%<*}
  ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$k" -s 1 -c 1 \
      -o $O/full_${n}_$TAG \
      python bench.py --L 512 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_${n}_$TAG.log 2>&1
done
echo done
