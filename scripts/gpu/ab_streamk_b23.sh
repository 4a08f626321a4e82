#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for r in 1 2 3; do
  BATCHES=5,4 PF_CTAS=-3 python scripts/time_prefill_ab.py
  BATCHES=5,4 python scripts/time_prefill_ab.py
done 2>&1 | tee gpurun_out/ab_streamk_b5.log
