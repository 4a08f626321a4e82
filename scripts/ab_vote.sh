#!/bin/bash
# A/B of the vote-first chunk max in the swapped decode consumers: libhpa.so vs variants/novote.so
timeout -s KILL 600 python -m pytest tests/test_gpu_fp8.py tests/test_gpu_parity.py -m gpu -x -q -k "decode or fp8" 2>&1 | tail -2
for r in 1 2; do
for lib in paper_2605_09100_b200/libhpa.so variants/novote.so; do
  echo "== $lib"
  HPA_LIB_PATH=$PWD/$lib timeout -s KILL 200 python scripts/time_fp8.py 2>&1 | tail -2
done
done
