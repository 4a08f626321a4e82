set -u
timeout -s KILL 200 python -c "import torch; torch.zeros(1).cuda(); print('warm')"
for pc in 1 2; do for c in c a; do echo "pieces=$pc"; HPA_CASC_PIECES=$pc CASE=$c timeout -s KILL 60 python -u scripts/dbg_cascade.py 2>&1 | tail -2; done; done
