#!/bin/bash
# A/B of variant builds: prefill (configs[2], B=4) and the decode step (configs[1]).
for lib in paper_2605_09100_b200/libhpa.so variants/*.so; do
  echo "== $lib"
  HPA_LIB_PATH=$PWD/$lib timeout -s KILL 120 python scripts/run_prefill.py --batch 4 --reps 4 2>&1 | tail -2
  HPA_LIB_PATH=$PWD/$lib timeout -s KILL 200 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-extra 2>&1 | tail -1 | python3 -c "
import sys,json
d=json.loads(sys.stdin.read()); print('decode step ms', d['ms_per_step'], 'decode call ms', d['roofline']['launch_ms'], 'frac', d['roofline']['frac'], 'clk', d['clocks']['sm_mhz'])"
done
