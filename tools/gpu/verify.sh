# Session start check: build, GPU tests, smoke, default bench line.
O=gpurun_out/verify; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "pytest rc $?" >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; echo "smoke rc $?" >> $O/smoke.log
tail -2 $O/smoke.log
timeout 900 python bench.py > $O/bench_default.log 2>&1; echo "rc $?" >> $O/bench_default.log
tail -c 1500 $O/bench_default.log
