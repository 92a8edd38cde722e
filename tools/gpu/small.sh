# small-panel TSQR of register leaves + colsum finish: GPU tests, cfg1 / cfg3 benches
O=gpurun_out/small; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc $?" >> $O/pytest_gpu.log
for r in 1 0; do RSVD_HQR_REGS=$r timeout 300 python bench.py --config 1 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > $O/bench_cfg1_regs$r.log 2>&1; done
timeout 600 python bench.py --config 3 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_cfg3.log 2>&1
