# Round-2 closing evidence: parity tests, smoke, default bench (config 3), reference arm.
set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?"
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; echo "bench rc $?"; tail -1 gpurun_out/bench_default.log
timeout 600 python bench.py --config 2 --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/bench_cfg2.log 2>&1; echo "bench2 rc $?"; tail -1 gpurun_out/bench_cfg2.log
timeout 600 python bench.py --config 1 --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/bench_cfg1.log 2>&1; echo "bench1 rc $?"; tail -1 gpurun_out/bench_cfg1.log
