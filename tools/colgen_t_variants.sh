O=gpurun_out
for v in 0 128 64 32; do
  echo "== SCV_COLGEN_T=$v"
  SCV_COLGEN_T=$v timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench ms/map', round(d['ms_per_step'],1), 'rt', '%.1e' % d['roundtrip_rel_err'], 'peak', round(d['peak_mem_gb'],1), {k: round(v,1) for k, v in d['stages_ms_per_step'].items() if v > 20})"
done
SCV_COLGEN_T=64 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "c4 or slab or streamed or orders or linear" 2>&1 | tail -2
