set -u
timeout -s KILL 200 python -c "import torch; torch.zeros(1).cuda(); print('warm')"
for c in lt tl t700; do CASE=$c timeout -s KILL 40 python -u scripts/dbg_f32.py 2>&1 | tail -1; done
timeout -s KILL 400 python -m pytest tests/test_gpu_fp8.py tests/test_gpu_fp8_edges.py tests/test_gpu_fuzz.py -q -p no:cacheprovider -x > gpurun_out/r2c_fp8.log 2>&1; echo "fp8+fuzz rc=$?"; tail -4 gpurun_out/r2c_fp8.log
SCRIPT=scripts/time_fp8.py ROUNDS=2 LIBS=variants/f32off.so bash scripts/ab_libs.sh 2>&1 | tee gpurun_out/r2c_fp8time.log
