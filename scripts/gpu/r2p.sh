set -u
timeout -s KILL 200 python -c "import torch; torch.zeros(1).cuda(); print('warm')"
timeout -s KILL 400 python -m pytest tests/test_gpu_fp8.py tests/test_gpu_fp8_edges.py tests/test_gpu_fuzz.py -q -p no:cacheprovider -x > gpurun_out/r2p_pytest.log 2>&1; echo "fp8 tests rc=$?"; tail -3 gpurun_out/r2p_pytest.log
SCRIPT=scripts/time_fp8.py ROUNDS=3 LIBS=variants/f32s8.so bash scripts/ab_libs.sh 2>&1 | grep fp8 | tee gpurun_out/r2p_ab.log
