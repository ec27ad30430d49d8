#!/bin/bash
O=gpurun_out; mkdir -p $O
SCV_LIB=variants/lib_stats.so timeout 200 python tools/pipe_stats.py 64 2>&1 | tail -5 > $O/r02r_pipe_stats.txt; cat $O/r02r_pipe_stats.txt | cut -c1-200
timeout 300 python tools/small_profile.py 64 300 2>&1 | head -45
