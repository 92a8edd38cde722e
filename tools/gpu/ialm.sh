# IALM update emitting M's slices: rrpca tests, cfg5 A/B
O=gpurun_out/ialm; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -k "rrpca" > $O/pytest_rrpca.log 2>&1; echo "pytest rc $?" >> $O/pytest_rrpca.log
for s in 1 0; do RSVD_IALM_SLICED=$s timeout 900 python bench.py --config 5 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_cfg5_sliced$s.log 2>&1; done
