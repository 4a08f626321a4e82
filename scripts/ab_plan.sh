#!/bin/bash
# planner constants sweep: main decode call, ragged, P=64, LMAG decode
for cfg in "1.5 8" "0.5 4" "4 8" "8 8" "1.5 20"; do
  set -- $cfg
  HPA_PLAN_C0=$1 HPA_PLAN_COMBINE=$2 timeout -s KILL 300 python bench.py --no-cpu-baseline > /tmp/abp.json 2>/tmp/abp.err
  python3 -c "
import json
try:
  d=json.loads(open('/tmp/abp.json').read().strip().splitlines()[-1]); v=d['decode_variants']
  print('c0=$1 comb=$2 main', d['roofline']['launch_ms'], 'ragged', v['ragged_U1K_8K']['decode_ms'], 'p64', v['page_size_64']['decode_ms'], 'lmag', d['lmag']['decode_ms'], 'shared', d['next']['shared_sets']['decode_ms'])
except Exception as e: print('FAILED', open('/tmp/abp.err').read()[-500:])"
done
