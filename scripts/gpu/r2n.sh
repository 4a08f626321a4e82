set -u
timeout -s KILL 200 python -c "import torch; torch.zeros(1).cuda(); print('warm')"
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_fp8.py tests/test_gpu_fp8_edges.py tests/test_gpu_append_decode.py tests/test_gpu_cascade.py tests/test_gpu_fork.py -q -p no:cacheprovider -x > gpurun_out/r2n_pytest.log 2>&1; echo "decode tests rc=$?"; tail -3 gpurun_out/r2n_pytest.log
SCRIPT=scripts/time_plan.py ROUNDS=3 LIBS=variants/wp0.so bash scripts/ab_libs.sh 2>&1 | grep bf16 | tee gpurun_out/r2n_ab.log
