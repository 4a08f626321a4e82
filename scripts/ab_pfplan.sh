#!/bin/bash
# prefill planner per-CTA overhead constant (key tiles), configs[2] B=1..3
for r in 1 2; do
for o in 3.3 2.0 5.0 8.0; do
  echo "== HPA_PF_OVH=$o"; HPA_PF_OVH=$o BATCHES=1,2,3 MODES=0 ROUNDS=1 timeout -s KILL 200 python scripts/time_prefill_split.py 2>&1 | grep "  B="
done
done
