echo "== probe"; OZ_TIMELINE=1 timeout 120 ./tools/test_ozaki_base 10000 5000 20 0 64 2>&1 | grep "trans\|us:"
timeout 120 ./tools/test_ozaki_base 20000 4000 10 0 128 2>&1 | grep "trans"
timeout 120 ./tools/test_ozaki_base 3000 1100 5 0 2>&1 | grep "trans"
timeout 300 python bench.py --config 2 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/la_cfg2.log 2>&1; echo rc $?
timeout 300 python bench.py --config 3 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/la_cfg3.log 2>&1; echo rc $?
timeout 300 python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/la_cfg5.log 2>&1; echo rc $?
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/la_pytest.log 2>&1; echo pytest rc $?
tail -3 gpurun_out/la_pytest.log
