#!/bin/bash
# (experiment record: the fused-merge build and its HPA_PF_SEP_MERGE knob were not kept; profiles/r2_prefill_fused_merge_ab.log)
# persistent prefill: split units merged after each CTA's item list by the last-arriving piece
# (default) vs the separate prefill_combine_kernel (HPA_PF_SEP_MERGE)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_prefill_split.py tests/test_gpu_fullsize.py -q -x -k "prefill" 2>&1 | tail -2
for r in 1 2 3; do
  BATCHES=1,2 python scripts/time_prefill_ab.py
  BATCHES=1,2 HPA_PF_SEP_MERGE=1 python scripts/time_prefill_ab.py
done 2>&1 | tee gpurun_out/ab_fused_merge.log
