#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
SCRIPT=scripts/time_variants.py LIBS="variants/early1.so variants/early3.so" ROUNDS=3 bash scripts/ab_libs.sh 2>&1 | tee gpurun_out/ab_early.log
