set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_cfg2.log 2>&1; echo "bench rc $?"
timeout 900 python bench.py --config 4 --steps 3 --warmup 3 > gpurun_out/bench_cfg4.log 2>&1; echo "bench4 rc $?"
tail -c 3000 gpurun_out/bench_cfg2.log; tail -c 3000 gpurun_out/bench_cfg4.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_cfg2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_cfg2.log 2>&1; echo "ncu rc $?"
