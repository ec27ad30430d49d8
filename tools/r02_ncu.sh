#!/bin/bash
# ncu --set full of the ring kernels (K = 2047) on a beta slab of L = 1024, plus the launch list of the
# default bench command; summaries only come back (profiles/ keeps them)
# usage: tools/r02_ncu.sh TAG [NB]
TAG=${1:-r02}; NB=${2:-64}
O=gpurun_out; mkdir -p $O /tmp/ncu
timeout 200 python tools/prof_slab.py 1024 $NB > $O/prof_slab_$TAG.log 2>&1 || { cat $O/prof_slab_$TAG.log; exit 1; }
for spec in "k_ana_colgen_p:1:1" "k_pfa_rows_p:2:2" "k_syn_gamma_qp:1:1"; do
  k=${spec%%:*}; rest=${spec#*:}; sk=${rest%%:*}; c=${rest#*:}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s $sk -c $c -f -o /tmp/ncu/full_${k}_$TAG \
    python tools/prof_slab.py 1024 $NB > $O/ncu_${k}_$TAG.log 2>&1
  { echo "== $k ($TAG, $NB beta rows of L=1024)";
    python tools/ncu_key.py /tmp/ncu/full_${k}_$TAG.ncu-rep;
    python tools/ncu_summary.py /tmp/ncu/full_${k}_$TAG.ncu-rep;
    echo "## per-source-line warp-stall samples (top 40)";
    python tools/ncu_lines.py /tmp/ncu/full_${k}_$TAG.ncu-rep 40; } > $O/ncu_sum_${k}_$TAG.txt 2>&1
done
# launch list of the bench command (per-launch times are cold-cache and serialised: shares only)
timeout 900 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/${TAG}_bench_plain.json 2>$O/${TAG}_bench_plain.err && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file $O/${TAG}_launches_L1024.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/${TAG}_ncu_bench.log 2>&1
python tools/summarize_launches.py $O/${TAG}_launches_L1024.csv > $O/${TAG}_launches_L1024_summary.txt 2>&1; tail -25 $O/${TAG}_launches_L1024_summary.txt
# other configurations for the record
timeout 600 python bench.py --real --no-cpu-baseline > $O/${TAG}_bench_real.json 2>$O/${TAG}_bench_real.err; tail -c 300 $O/${TAG}_bench_real.json
timeout 600 python bench.py --L 512 --jmin 2 --no-cpu-baseline > $O/${TAG}_bench_c3.json 2>$O/${TAG}_bench_c3.err
timeout 600 python bench.py --L 128 --spin 2 --jmin 2 --no-cpu-baseline > $O/${TAG}_bench_c2.json 2>$O/${TAG}_bench_c2.err
timeout 600 python bench.py --L 64 --jmin 2 --no-cpu-baseline > $O/${TAG}_bench_c1.json 2>$O/${TAG}_bench_c1.err
timeout 1200 python bench.py --streamed --L 2048 --spin 2 --jmin 4 --no-cpu-baseline --steps 2 --warmup 1 > $O/${TAG}_bench_c5.json 2>$O/${TAG}_bench_c5.err
for f in real c3 c2 c1 c5; do python -c "
import json; d=json.loads(open('$O/${TAG}_bench_$f.json').read().strip().splitlines()[-1]); print('$f', d['config'].get('workload'), round(d['value'],4), d['unit'], round(d['ms_per_step'],2), 'ms rt', d.get('roundtrip_rel_err'), 'first map', round(d.get('first_map_ms',0)))" 2>&1 | tail -1; done
ls -la $O
