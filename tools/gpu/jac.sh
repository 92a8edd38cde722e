timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py -q -p no:cacheprovider -x > gpurun_out/jac_pytest.log 2>&1; echo pytest rc $?; tail -3 gpurun_out/jac_pytest.log
for c in 2 3 1; do timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/jac_cfg$c.log 2>&1; echo cfg$c rc $?; done
