# exponent blocks 4096 (FP64) / 8192 (FP32): full GPU tests, cfg3 / cfg4 / cfg2 benches
O=gpurun_out/et2; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc $?" >> $O/pytest_gpu.log
for c in 3 4 2; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_cfg$c.log 2>&1; done
