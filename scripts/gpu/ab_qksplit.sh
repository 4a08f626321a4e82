#!/bin/bash
# (experiment record: the HPA_QK_SPLIT build was not kept; profiles/r2_prefill_qk_split_ab.log)
# prefill: Q K^T as two N = 64 halves with separate commits (HPA_QK_SPLIT) vs the default
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
HPA_LIB_PATH=$PWD/variants/qksplit.so timeout 600 python -m pytest tests/test_gpu_prefill_split.py tests/test_gpu_parity.py -q -x -k "prefill" 2>&1 | tail -2
PF_CTAS=-3 BATCHES=4,1 SCRIPT=scripts/time_prefill_ab.py LIBS="variants/qksplit.so" ROUNDS=3 bash scripts/ab_libs.sh 2>&1 | tee gpurun_out/ab_qksplit.log
