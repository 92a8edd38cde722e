# balanced double-buffered panel apply (Np = 128): GPU tests, A/B benches
O=gpurun_out/apply; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc $?" >> $O/pytest_gpu.log
for c in 3 4; do for a in 1 0; do
  RSVD_APPLY128=$a timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_cfg${c}_apply$a.log 2>&1
done; done
