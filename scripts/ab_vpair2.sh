#!/bin/bash
# A/B of the fp8 V pair-row layout: working tree (libhpa.so) vs HEAD build (variants/headvpair.so)
timeout -s KILL 500 python -m pytest tests/test_gpu_fp8.py -m gpu -x -q 2>&1 | tail -3
for r in 1 2; do
for lib in paper_2605_09100_b200/libhpa.so variants/headvpair.so; do
  echo "== $lib"
  HPA_LIB_PATH=$PWD/$lib timeout -s KILL 200 python scripts/time_fp8.py 2>&1 | tail -2
done
done
