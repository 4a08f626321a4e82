#!/bin/bash
# Interleaved A/B over the default build and variant libraries: ROUNDS x (each lib) of SCRIPT.
# LIBS (space-separated, default variants/*.so) selects the variants.
SCRIPT=${SCRIPT:-scripts/time_prefill_ab.py}
LIBS=${LIBS:-$(ls variants/*.so 2>/dev/null)}
for r in $(seq ${ROUNDS:-3}); do
  for lib in paper_2605_09100_b200/libhpa.so $LIBS; do
    HPA_LIB_PATH=$PWD/$lib timeout -s KILL 300 python $SCRIPT 2>&1 | tail -2
  done
done
