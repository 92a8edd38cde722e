timeout 300 ./tools/bench_jacobi > gpurun_out/jblk_bench.log 2>&1; echo "rc $?" >> gpurun_out/jblk_bench.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/jblk_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/jblk_pytest.log
for c in 2 3 1; do timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/jblk_cfg$c.log 2>&1; done
