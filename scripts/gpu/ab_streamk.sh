#!/bin/bash
# configs[2] prefill: default (stream-K persistent under 4 waves) vs one CTA per item (-3)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for r in 1 2 3; do
  python scripts/time_prefill_ab.py
  PF_CTAS=-3 python scripts/time_prefill_ab.py
done 2>&1 | tee gpurun_out/ab_streamk.log
python -m pytest tests/test_gpu_prefill_split.py tests/test_gpu_fuzz.py tests/test_gpu_fullsize.py tests/test_gpu_parity.py -q -x 2>&1 | tail -3
