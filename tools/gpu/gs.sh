# symmetric Gram (Ng = 128) + register-held Householder vectors (RPL <= 16): GPU tests, A/B benches, graph probe
O=gpurun_out/gs; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc $?" >> $O/pytest_gpu.log
for c in 3 4; do for s in 1 0; do
  RSVD_GRAM_SYM=$s timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_cfg${c}_sym$s.log 2>&1
done; done
timeout 300 python bench.py --config 1 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > $O/bench_cfg1.log 2>&1
timeout 300 python tools/graph_vs_eager.py > $O/graph.log 2>&1
