# r2 session 3: F32 fp8 decode hang hunt + SM_SEQ prefill A/B
set -u
mkdir -p gpurun_out
timeout -s KILL 200 python -c "import torch; torch.zeros(1).cuda(); print('warm')"
for lib in paper_2605_09100_b200/libhpa.so variants/dbgring.so; do
  ls -la $lib
  HPA_LIB_PATH=$PWD/$lib timeout -s KILL 90 python -u -m pytest tests/test_gpu_fp8.py -q -s -p no:cacheprovider -x -k "decode" > gpurun_out/r2a_fp8_$(basename $lib).log 2>&1; echo "$lib fp8 decode rc=$?"; tail -8 gpurun_out/r2a_fp8_$(basename $lib).log
done
timeout -s KILL 300 python -u -m pytest tests/test_gpu_prefill_split.py tests/test_gpu_fuzz.py -q -p no:cacheprovider -x -k "prefill" > gpurun_out/r2a_prefill.log 2>&1; echo "prefill tests rc=$?"; tail -4 gpurun_out/r2a_prefill.log
ROUNDS=2 LIBS=variants/smseq0.so bash scripts/ab_libs.sh 2>&1 | tee gpurun_out/r2a_ab.log
SCRIPT=scripts/time_fp8.py ROUNDS=1 LIBS=variants/f32off.so bash scripts/ab_libs.sh 2>&1 | tee gpurun_out/r2a_fp8time.log
