#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
export PF_CTAS=-3
SCRIPT=scripts/time_prefill_ab.py LIBS="${LIBS:-variants/l2pf2.so variants/l2pf4.so variants/l2pf8.so}" ROUNDS=3 bash scripts/ab_libs.sh 2>&1 | tee gpurun_out/ab_l2pf.log
