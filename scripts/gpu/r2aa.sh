set -u
timeout -s KILL 200 python -c "import torch; torch.zeros(1).cuda(); print('warm')"
for r in 1 2; do for c0 in 0.5 1.5 3.0 4.0; do HPA_PLAN_C0=$c0 timeout 120 python scripts/time_plan.py | cut -c1-60; done; done 2>&1 | grep -v Warn
