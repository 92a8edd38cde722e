timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/slc2_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/slc2_pytest.log
for c in 3 2; do timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/slc2_cfg$c.log 2>&1; done
