#!/bin/bash
# usage: tools/regs.sh file.cu [grep-pattern] [nvcc defines...]
f=$1; pat=${2:-.}; shift; shift
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -Xptxas -v -c "$f" -o /tmp/regs_$$.o "$@" 2>&1 | python3 -c "
import sys,re
cur=None; st=sp='?'
for line in sys.stdin:
    if 'error' in line: print(line.rstrip())
    m=re.search(r\"Compiling entry function '(\S+)'\",line)
    if m: cur=m.group(1); continue
    m=re.search(r'(\d+) bytes stack frame, (\d+) bytes spill stores',line)
    if m and cur: st=m.group(1); sp=m.group(2)
    m=re.search(r'Used (\d+) registers',line)
    if m and cur:
        print(f'{cur[:50]:50s} regs={m.group(1)} stack={st} spill={sp}'); cur=None
" | sort | grep -E "$pat"
rm -f /tmp/regs_$$.o
