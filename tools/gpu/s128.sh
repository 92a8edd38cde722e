# FP32 Ozaki single-CTA N=128 vs the column-pair launch
O=gpurun_out/s128; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "fp32 or config4" > $O/pytest_fp32.log 2>&1; echo "pytest rc $?" >> $O/pytest_fp32.log
timeout 600 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_cfg4_single.log 2>&1; echo "rc $?" >> $O/bench_cfg4_single.log
RSVD_OZ_SINGLE128=0 timeout 600 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_cfg4_pair.log 2>&1; echo "rc $?" >> $O/bench_cfg4_pair.log
