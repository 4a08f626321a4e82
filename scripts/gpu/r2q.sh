set -u
timeout -s KILL 200 python -c "import torch; torch.zeros(1).cuda(); print('warm')"
timeout -s KILL 400 python -m pytest tests/test_gpu_cascade.py -q -p no:cacheprovider -x > gpurun_out/r2q_pytest.log 2>&1; echo "cascade tests rc=$?"; tail -3 gpurun_out/r2q_pytest.log
for r in 1 2; do for lib in paper_2605_09100_b200/libhpa.so variants/cs8.so variants/cs10.so; do echo "== $lib"; CASES=64:16384:1024,64:4096:1024,64:1024:1024,16:16384:4096,64:16384:64 HPA_LIB_PATH=$PWD/$lib python scripts/time_cascade.py; done; done 2>&1 | tee gpurun_out/r2q_ab.log
