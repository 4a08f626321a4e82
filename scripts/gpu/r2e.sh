set -u
timeout -s KILL 200 python -c "import torch; torch.zeros(1).cuda(); print('warm')"
for r in 1 2; do for c0 in 0.5 1.0 1.5 2.5; do echo "C0=$c0"; HPA_PLAN_C0=$c0 python scripts/time_fp8.py; done; done 2>&1 | tee gpurun_out/r2e_c0.log
