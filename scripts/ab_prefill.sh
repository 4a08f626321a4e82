#!/bin/bash
for lib in paper_2605_09100_b200/libhpa.so $(ls variants/*.so 2>/dev/null); do
  echo "== $lib"
  HPA_LIB_PATH=$PWD/$lib timeout -s KILL 120 python scripts/run_prefill.py --batch 4 --reps 4 2>&1 | tail -2
  HPA_LIB_PATH=$PWD/$lib timeout -s KILL 120 python scripts/run_prefill.py --batch 1 --reps 4 2>&1 | tail -1
done
