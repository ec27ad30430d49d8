#!/bin/bash
# usage: tools/spills.sh file.cu kernel-substring [nvcc defines...]  -> local-memory ops by source line
f=$1; k=$2; shift 2
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -lineinfo -cubin -o /tmp/spills.cubin "$f" "$@" 2>/dev/null
/usr/local/cuda/bin/nvdisasm --print-line-info /tmp/spills.cubin > /tmp/spills.sass 2>&1
python3 - "$k" <<'PY'
import sys, collections
k = sys.argv[1]
for sec in open('/tmp/spills.sass').read().split('//--------------------- .text.'):
    if k in sec[:300]:
        loc = None; c = collections.Counter()
        for line in sec.splitlines():
            if '//## File' in line: loc = line.split('/')[-1]
            if 'STL' in line or 'LDL' in line: c[loc] += 1
        for kk, v in c.most_common(15): print(v, kk)
        break
PY
