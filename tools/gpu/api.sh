timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/api_pytest.log 2>&1; echo pytest rc $?
tail -15 gpurun_out/api_pytest.log
timeout 300 python bench.py --config 2 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/api_cfg2.log 2>&1; echo rc $?
timeout 300 python bench.py --config 1 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/api_cfg1.log 2>&1; echo rc $?
