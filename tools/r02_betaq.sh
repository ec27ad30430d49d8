#!/bin/bash
# GEMM build of the beta-quadrature table vs the direct build; then the parity tests that go through the table
O=gpurun_out; mkdir -p $O
timeout 600 python tools/betaq_check.py 128 256 512 1024 2>&1 | tail -6
timeout 900 python -m pytest tests/test_gpu_parity_full.py -m gpu -x -q -k "quadrature or thresholded or forward_slab" 2>&1 | tail -3
