#!/bin/bash
for S in 0 2 6 7 13 20; do
  timeout -s KILL 200 python bench.py --steps 100 --warmup 10 --no-cpu-baseline --no-extra --splits $S 2>&1 | tail -1 | python3 -c "
import sys,json
d=json.loads(sys.stdin.read()); print('splits $S: decode call ms', d['roofline']['launch_ms'], 'GB/s', d['roofline']['achieved'])"
done
