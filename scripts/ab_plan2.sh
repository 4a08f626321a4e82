#!/bin/bash
# decode planner constants, configs[1] decode call only (scripts/time_fp8.py bf16 line), 2 rounds
for r in 1 2; do
for cfg in "0.5 4" "0.25 4" "0.1 4" "0.25 2" "0.1 1" "1.0 4"; do
  set -- $cfg
  echo -n "c0=$1 comb=$2 "; HPA_PLAN_C0=$1 HPA_PLAN_COMBINE=$2 timeout -s KILL 200 python scripts/time_fp8.py 2>&1 | grep bf16
done
done
