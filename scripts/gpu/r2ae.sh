set -u
timeout -s KILL 200 python -c "import torch; torch.zeros(1).cuda(); print('warm')"
for r in 1 2; do for f in none 0.5:2 1:2 2:2 1:4; do if [ $f = none ]; then python scripts/time_plan.py | cut -c1-62 | sed "s/^/FINE=none /"; else HPA_PLAN_FINE=$f python scripts/time_plan.py | cut -c1-62 | sed "s/^/FINE=$f /"; fi; done; done 2>&1 | grep FINE
