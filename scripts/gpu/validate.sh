# GPU validation: the full -m gpu suite (no -x: list every failure), then the bench.
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests/test_gpu_fp8_edges.py tests/test_gpu_head_shard.py tests/test_gpu_parity.py::test_split_invariance_fp32_partials "tests/test_gpu_fullsize.py::test_prefill_config2_b4_full_size_sampled_clusters" -q -p no:cacheprovider > gpurun_out/pytest_new.log 2>&1; echo "new tests rc=$?"
tail -15 gpurun_out/pytest_new.log
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -8 gpurun_out/pytest_gpu.log
if [ "${RUN_BENCH:-0}" = 1 ]; then timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; fi
