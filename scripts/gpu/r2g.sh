set -u
timeout -s KILL 200 python -c "import torch; torch.zeros(1).cuda(); print('warm')"
for r in 1 2; do for c0 in 3.0 4.0 5.0 6.0 8.0 12.0 20.0; do HPA_PLAN_C0=$c0 timeout 120 python scripts/time_plan.py; done; done 2>&1 | grep -v Warn | tee gpurun_out/r2g_c0.log
