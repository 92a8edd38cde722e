# tensor peaks, bench default (cfg3) with cpu baseline + e2e, cfg2, bench contract test
./tools/peaks_tc > gpurun_out/peaks_tc.json 2>&1; echo peaks rc $?; cat gpurun_out/peaks_tc.json
timeout 900 python bench.py > gpurun_out/b_cfg3.log 2>&1; echo cfg3 rc $?
timeout 600 python bench.py --config 2 --steps 50 --warmup 5 > gpurun_out/b_cfg2.log 2>&1; echo cfg2 rc $?
timeout 600 python bench.py --config 1 --steps 50 --warmup 5 > gpurun_out/b_cfg1.log 2>&1; echo cfg1 rc $?
timeout 900 python bench.py --config 5 --steps 3 --warmup 3 > gpurun_out/b_cfg5.log 2>&1; echo cfg5 rc $?
timeout 900 python -m pytest tests/test_bench_contract.py tests/test_gpu_api.py -q -p no:cacheprovider > gpurun_out/b_pytest.log 2>&1; echo pytest rc $?
tail -3 gpurun_out/b_pytest.log
