# quick GPU validation: parity tests + default bench + launch list of one step
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 50 --warmup 5 > gpurun_out/bench_cfg2.log 2>&1; echo "bench rc $?"
tail -c 1500 gpurun_out/bench_cfg2.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"rsvd|gemm|chol|gram|panel|jacobi|omega|hqr|tsqr|ozaki" --csv --log-file gpurun_out/launches_cfg2.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_cfg2.log 2>&1; echo "ncu rc $?"
