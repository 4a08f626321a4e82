#!/bin/bash
# (experiment record: the multi-row combine build was not kept; profiles/r2_prefill_combine_rows_ab.log)
# prefill split merge: rows per warp of the combine kernel (HPA_PF_COMBINE_ROWS; 1 = one row per warp)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_prefill_split.py tests/test_gpu_fullsize.py tests/test_gpu_fuzz.py -q -x -k "prefill" 2>&1 | tail -2
BATCHES=1,2 SCRIPT=scripts/time_prefill_ab.py LIBS="variants/crows1.so variants/crows4.so variants/crows16.so" ROUNDS=3 bash scripts/ab_libs.sh 2>&1 | tee gpurun_out/ab_combine_rows.log
