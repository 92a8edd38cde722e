timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/fused_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/fused_pytest.log
for c in 2 3 1; do timeout 600 python bench.py --config $c --steps 30 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/fused_cfg$c.log 2>&1; done
