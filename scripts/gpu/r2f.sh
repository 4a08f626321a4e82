set -u
timeout -s KILL 200 python -c "import torch; torch.zeros(1).cuda(); print('warm')"
for r in 1 2; do for c0 in 0.5 0.75 1.0 1.25 1.5 2.0 3.0; do HPA_PLAN_C0=$c0 timeout 120 python scripts/time_plan.py; done; done 2>&1 | grep -v Warn | tee gpurun_out/r2f_c0.log
for cb in 2.0 8.0; do HPA_PLAN_C0=1.0 HPA_PLAN_COMBINE=$cb timeout 120 python scripts/time_plan.py; done 2>&1 | tee -a gpurun_out/r2f_c0.log
