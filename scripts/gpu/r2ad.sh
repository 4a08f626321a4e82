set -u
timeout -s KILL 200 python -c "import torch; torch.zeros(1).cuda(); print('warm')"
for lib in paper_2605_09100_b200/libhpa.so variants/cs3.so variants/cs4.so; do
  HPA_LIB_PATH=$PWD/$lib timeout -s KILL 300 python -m pytest tests/test_gpu_cascade.py -q -p no:cacheprovider -x > gpurun_out/r2ad_$(basename $lib).log 2>&1; echo "$lib tests rc=$?"; tail -1 gpurun_out/r2ad_$(basename $lib).log
done
for r in 1 2; do for lib in paper_2605_09100_b200/libhpa.so variants/cs3.so variants/cs4.so; do echo "== $lib"; CASES=64:16384:1024,64:4096:1024,64:1024:1024,16:16384:4096,64:16384:64 HPA_LIB_PATH=$PWD/$lib python scripts/time_cascade.py | cut -c1-80; done; done
