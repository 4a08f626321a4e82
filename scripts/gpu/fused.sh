set -u
python -m pytest tests/test_gpu_append_decode.py -q -p no:cacheprovider -x > gpurun_out/pytest_fused.log 2>&1; echo "fused tests rc=$?"; tail -15 gpurun_out/pytest_fused.log
timeout 300 python scripts/time_step_fused.py > gpurun_out/time_step_fused.log 2>&1; echo "timing rc=$?"; cat gpurun_out/time_step_fused.log
timeout 600 python bench.py --no-extra --no-cpu-baseline > gpurun_out/bench_fused.json 2> gpurun_out/bench_fused.err; echo "bench rc=$?"; head -c 2500 gpurun_out/bench_fused.json; tail -3 gpurun_out/bench_fused.err
