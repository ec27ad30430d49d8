#!/bin/bash
# per-role pipeline counters of stats builds (variants/lib_stats.so and any variants/lib_*exp*.so / lib_gq*.so)
for f in variants/lib_stats.so variants/lib_gq*.so variants/lib_*exp*.so; do [ -f $f ] || continue; echo "== $f"; SCV_LIB=$f timeout 200 python tools/pipe_stats.py 32 2>&1 | grep -v "^colgen\|^rows" | cut -c1-230; done
