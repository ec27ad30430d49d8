#!/bin/bash
O=gpurun_out; mkdir -p $O /tmp/ncu
for k in k_sht_contract_w k_sht_bins_w; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 -f -o /tmp/ncu/sht_$k python tools/sht_prof.py 1024 > $O/ncu_sht_$k.log 2>&1
  { echo "== $k"; python tools/ncu_key.py /tmp/ncu/sht_$k.ncu-rep; python tools/ncu_summary.py /tmp/ncu/sht_$k.ncu-rep | grep -E "Throughput|Hit Rate|Issue|stall|Duration|Warps"; echo "## lines"; python tools/ncu_lines.py /tmp/ncu/sht_$k.ncu-rep 12; } > $O/r03_ncu_$k.txt 2>&1
  head -60 $O/r03_ncu_$k.txt
done
