O=gpurun_out
python tools/prof_slab.py 1024 16 > $O/ps.log 2>&1 || { cat $O/ps.log; exit 1; }
for k in k_ana_colgen k_pfa_rows k_syn_alpha k_syn_gamma_q; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 -o $O/prof_${k}_2047 python tools/prof_slab.py 1024 16 > $O/ncu_$k.log 2>&1
done
ls $O
