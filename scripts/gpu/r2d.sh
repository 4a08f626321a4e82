set -u
timeout -s KILL 200 python -c "import torch; torch.zeros(1).cuda(); print('warm')"
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_fp8.py tests/test_gpu_fp8_edges.py tests/test_gpu_append_decode.py tests/test_gpu_fork.py tests/test_gpu_head_shard.py -q -p no:cacheprovider -x > gpurun_out/r2d_pytest.log 2>&1; echo "decode tests rc=$?"; tail -4 gpurun_out/r2d_pytest.log
SCRIPT=scripts/time_fp8.py ROUNDS=3 LIBS=variants/base.so bash scripts/ab_libs.sh 2>&1 | tee gpurun_out/r2d_ab.log
for c0 in 0.25 0.5 1.0; do echo "C0=$c0"; HPA_PLAN_C0=$c0 python scripts/time_fp8.py; done 2>&1 | tee gpurun_out/r2d_c0.log
