#!/bin/bash
# full GPU suite + default bench on the current build
O=gpurun_out; mkdir -p $O; TAG=${1:-r02x}
timeout 2400 python -m pytest tests -m gpu -x -q > $O/${TAG}_pytest_gpu.log 2>&1; tail -3 $O/${TAG}_pytest_gpu.log
timeout 900 python bench.py > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err; python -c "
import json; d=json.loads(open('$O/${TAG}_bench.json').read().strip().splitlines()[-1]); print('C4', d['value'], 'maps/s', d['ms_per_step'], 'ms; e2e', d['e2e']['value'], 'first map', d['first_map_ms'], 'paper frac', d['paper_roofline']['frac'], 'roofline', d['roofline']['stage'], d['roofline']['frac'])"
