#!/bin/bash
# (experiment record: the HPA_PFUSED_COMBINE build was not kept; profiles/r2_decode_fused_combine_ab.log)
# persistent decode: a5 fused into the kernel (HPA_PFUSED_COMBINE) vs the separate combine kernel
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
HPA_LIB_PATH=$PWD/variants/pfc.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_append_decode.py tests/test_gpu_fp8.py tests/test_gpu_fuzz.py tests/test_gpu_cascade.py tests/test_gpu_fullsize.py -q -x -p no:cacheprovider 2>&1 | tail -2
SCRIPT=scripts/time_plan.py LIBS="variants/pfc.so" ROUNDS=4 bash scripts/ab_libs.sh 2>&1 | tee gpurun_out/ab_pfc.log
