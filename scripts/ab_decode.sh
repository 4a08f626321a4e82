#!/bin/bash
for lib in paper_2605_09100_b200/libhpa.so $(ls variants/*.so 2>/dev/null); do
  echo "== $lib"
  for r in 1 2; do
  HPA_LIB_PATH=$PWD/$lib timeout -s KILL 200 python bench.py --steps 100 --warmup 10 --no-cpu-baseline --no-extra 2>&1 | tail -1 | python3 -c "
import sys,json
d=json.loads(sys.stdin.read()); print('decode step ms', d['ms_per_step'], 'decode call ms', d['roofline']['launch_ms'], 'frac', d['roofline']['frac'], 'clk', d['clocks']['sm_mhz'])"
  done
done
