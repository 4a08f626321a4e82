# ncu --set full captures of the current kernels for profiles/ (traffic + summaries)
set -u
python scripts/ncu_step.py && ncu --set full --clock-control none --import-source on -k regex:decode_persistent -s 4 -c 1 -o gpurun_out/step_dec python scripts/ncu_step.py > gpurun_out/ncu_step.log 2>&1; echo "step rc=$?"
python scripts/run_prefill.py --batch 4 --reps 2 && ncu --set full --clock-control none --import-source on -k regex:prefill_kernel -s 1 -c 1 -o gpurun_out/pf4 python scripts/run_prefill.py --batch 4 --reps 2 > gpurun_out/ncu_pf4.log 2>&1; echo "pf4 rc=$?"
python scripts/ncu_fp8_decode.py && ncu --set full --clock-control none --import-source on -k regex:decode_persistent -s 3 -c 1 -o gpurun_out/fp8ef python scripts/ncu_fp8_decode.py > gpurun_out/ncu_fp8ef.log 2>&1; echo "fp8 rc=$?"
