#!/bin/bash
# decode call time vs forced split count, for the in-tree library and every variants/*.so
for lib in paper_2605_09100_b200/libhpa.so $(ls variants/*.so 2>/dev/null); do
  echo "== $lib"
  for S in ${SPLITS:-0 2 6 8 13}; do
    HPA_LIB_PATH=$PWD/$lib timeout -s KILL 200 python bench.py --steps 100 --warmup 10 --no-cpu-baseline --no-extra --splits $S > /tmp/abs.json 2>/tmp/abs.err
    python3 -c "
import sys,json
try:
  d=json.loads(open('/tmp/abs.json').read().strip().splitlines()[-1]); print('splits $S: decode call ms', d['roofline']['launch_ms'], 'GB/s', d['roofline']['achieved'])
except Exception as e: print('splits $S: FAILED', open('/tmp/abs.err').read()[-600:])"
  done
done
