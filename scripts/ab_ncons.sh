for lib in paper_2605_09100_b200/libhpa.so variants/c10s20.so variants/c5s10.so; do
  echo "== $lib"
  for r in 1 2; do HPA_LIB_PATH=$PWD/$lib timeout -s KILL 200 python scripts/time_fp8.py 2>&1 | tail -2; done
done
for lib in variants/c10s20.so variants/c5s10.so; do
  echo "== tests $lib"
  HPA_LIB_PATH=$PWD/$lib timeout -s KILL 400 python -m pytest tests/test_gpu_fp8.py tests/test_gpu_parity.py -m gpu -x -q -k "decode or fp8" 2>&1 | tail -2
done
