#!/bin/bash
# Long all-API fuzz on the GPU box: bf16 and fp8 token pages (each check decodes with cascade
# planner / forced / off; decode_partial and fused steps run with planner or forced cascade), and
# the cascade kernel variant for every call (HPA_FORCE_CS).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/fuzz_build.log 2>&1 || { tail gpurun_out/fuzz_build.log; exit 1; }
S=${SEEDS:-0,1,2,3,4,5,6,7}; O=${OPS:-600}
run() { local tag=$1; shift; env "$@" SEEDS=$S OPS=$O timeout 900 python scripts/fuzz_all.py > gpurun_out/fuzz_$tag.log 2>&1; echo "$tag rc=$?"; grep -v "^  " gpurun_out/fuzz_$tag.log | tail -12; }
run bf16 X=1
run fp8 FP8=1
run bf16_cs HPA_FORCE_CS=1
