O=gpurun_out
bash tools/ncu_pfa.sh 2047
python bench.py --L 512 --steps 1 --warmup 2 --no-cpu-baseline --no-e2e > $O/b512.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_ana_colgen -s 2 -c 1 -o $O/prof_colgen1023 python bench.py --L 512 --steps 1 --warmup 2 --no-cpu-baseline --no-e2e > $O/ncu_colgen.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_syn_gamma_q -s 20 -c 1 -o $O/prof_gq1023 python bench.py --L 512 --steps 1 --warmup 2 --no-cpu-baseline --no-e2e > $O/ncu_gq.log 2>&1
ls $O
