# FP32 exponent blocks of 4096 rows (drain every 64 units): probe check + timing, FP32 tests, cfg4 bench
O=gpurun_out/et; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
OZ_F32=1 timeout 120 ./tools/test_ozaki_base 9000 5000 0 0 128 > $O/check.log 2>&1; echo "rc $?" >> $O/check.log
OZ_F32=1 OZ_NOCHECK=1 timeout 120 ./tools/test_ozaki_base 250000 10000 5 0 128 2>&1 | grep trans > $O/probe.log
timeout 900 python -m pytest tests -m gpu -q -k "fp32 or config4" > $O/pytest.log 2>&1; echo "pytest rc $?" >> $O/pytest.log
timeout 600 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_cfg4.log 2>&1
