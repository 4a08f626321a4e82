set -u
timeout -s KILL 200 python -c "import torch; torch.zeros(1).cuda(); print('warm')"
for k in 1.75 1.4 1.1; do echo "== kappa $k"; HPA_CASC_MIN_SAVED=0 HPA_CASC_KAPPA=$k CASES=64:16384:1024,64:4096:1024,64:1024:1024,16:16384:4096,64:16384:64,32:2048:4096,64:512:4096,64:1024:4096,256:1024:4096 python scripts/time_cascade.py; done 2>&1 | tee gpurun_out/r2r.log
HPA_CASC_MIN_SAVED=0 python scripts/time_next.py 2>&1 | grep -A8 shared_sets | tee -a gpurun_out/r2r.log
