# Full GPU evidence run: build, parity tests, bench all configs, ncu launch
# list + full capture of the dominant pass kernels (cfg2).  Outputs in gpurun_out/.
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"
tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?"
timeout 600 python bench.py --steps 100 --warmup 10 > gpurun_out/bench_cfg2.log 2>&1; echo "bench2 rc $?"
for c in 1 3 5; do timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg$c.log 2>&1; echo "bench$c rc $?"; done
timeout 900 python bench.py --config 4 --steps 3 --warmup 3 > gpurun_out/bench_cfg4.log 2>&1; echo "bench4 rc $?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc $?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"rsvd|gemm|chol|gram|panel|jacobi|omega|hqr|tsqr|ozaki" --csv --log-file gpurun_out/launches_cfg2.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_cfg2.log 2>&1; echo "ncu launches rc $?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:ozaki_pass_kernel -s 12 -c 2 -o gpurun_out/ozaki_cfg2_full python bench.py --steps 1 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc $?"
