#!/bin/bash
# r02 GPU pass 4: pipelined row kernel -- accuracy, timings, variants, bench
O=gpurun_out; mkdir -p $O
timeout 300 python tools/fftbench.py 2047 > $O/r02d_fft.txt 2>&1
cat $O/r02d_fft.txt
: > $O/r02d_stage.txt
timeout 120 python tools/stagebench.py 2047 >> $O/r02d_stage.txt 2>&1
for f in variants/lib_*.so; do SCV_LIB=$f timeout 120 python tools/stagebench.py 2047 >> $O/r02d_stage.txt 2>&1; done
cat $O/r02d_stage.txt
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/r02d_bench.json 2> $O/r02d_bench.err
python -c "
import json; d=json.loads(open('$O/r02d_bench.json').read().strip().splitlines()[-1]); print('ms/map', d['ms_per_step'], 'rt', d['roundtrip_rel_err']); print({k: round(v,1) for k,v in d['stages_ms_per_step'].items() if v>1})"
for v in ng5 nio2 nbw2; do SCV_LIB=variants/lib_$v.so timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v ms/map', d['ms_per_step'], 'rt', d['roundtrip_rel_err']); print({k: round(v,1) for k,v in d['stages_ms_per_step'].items() if v>1})"; done
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "not 2048 and not c5" > $O/r02d_pytest.log 2>&1; tail -3 $O/r02d_pytest.log
