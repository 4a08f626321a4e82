set -u
timeout -s KILL 120 python -m pytest tests/test_gpu_fp8.py -q -p no:cacheprovider -x -k "decode" > gpurun_out/f32_t1.log 2>&1; echo "fp8 decode tests rc=$?"; tail -5 gpurun_out/f32_t1.log
timeout -s KILL 120 env HPA_LIB_PATH=$PWD/variants/f32off.so python -m pytest tests/test_gpu_fp8.py -q -p no:cacheprovider -x -k "decode" > gpurun_out/f32_t2.log 2>&1; echo "f32off decode tests rc=$?"; tail -3 gpurun_out/f32_t2.log
