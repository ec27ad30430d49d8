set -x
O=gpurun_out
./tools/micro/dmma > $O/dmma.txt 2>&1
timeout 300 python tools/fftbench.py 1023,2047 > $O/fftbench.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_pfa_rows -s 2 -c 1 -o $O/full_pfa_rows2047 python tools/fftbench.py 2047 > $O/ncu_rows2047.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_pfa_rows -s 2 -c 1 -o $O/full_pfa_rows1023 python tools/fftbench.py 1023 > $O/ncu_rows1023.log 2>&1
ls -la $O
