set -u
timeout -s KILL 200 python -c "import torch; torch.zeros(1).cuda(); print('warm')"
for r in 1 2; do
  python scripts/time_plan.py | cut -c1-60 | sed 's/^/default /'
  HPA_LIB_PATH=$PWD/variants/p9.so python scripts/time_plan.py | cut -c1-60 | sed 's/^/p9 /'
  for cb in 1.0 8.0; do HPA_PLAN_COMBINE=$cb python scripts/time_plan.py | cut -c1-60; done
  for c0 in 2.0 4.0; do HPA_PLAN_C0=$c0 python scripts/time_plan.py | cut -c1-60; done
done 2>&1 | grep -v Warn
