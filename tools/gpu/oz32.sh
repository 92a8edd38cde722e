# FP32 Ozaki (3-digit) path: parity tests, cfg4 bench (ozaki vs tf32)
O=gpurun_out/oz32; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "fp32 or config4" > $O/pytest_fp32.log 2>&1; echo "pytest rc $?" >> $O/pytest_fp32.log
timeout 600 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_cfg4_oz.log 2>&1; echo "rc $?" >> $O/bench_cfg4_oz.log
RSVD_FP32_PATH=tf32 timeout 600 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_cfg4_tf32.log 2>&1; echo "rc $?" >> $O/bench_cfg4_tf32.log
timeout 600 python bench.py --config 3 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_cfg3.log 2>&1; echo "rc $?" >> $O/bench_cfg3.log
