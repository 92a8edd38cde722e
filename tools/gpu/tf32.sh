timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "fp32 or config4_full_size_vs" > gpurun_out/tf32_pytest.log 2>&1; echo pytest rc $?; tail -3 gpurun_out/tf32_pytest.log
timeout 900 python bench.py --config 4 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/tf32_cfg4.log 2>&1; echo rc $?
