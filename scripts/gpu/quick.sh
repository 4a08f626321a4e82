python -m pytest tests/test_gpu_fork.py -q -p no:cacheprovider -x > gpurun_out/pytest_fork.log 2>&1; echo "fork tests rc=$?"; tail -25 gpurun_out/pytest_fork.log
python scripts/time_bench_loop.py > gpurun_out/bench_loop.log 2>&1; echo "bench loop rc=$?"; cat gpurun_out/bench_loop.log
