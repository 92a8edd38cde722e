# FP32 row-pair (cta_group::2) Ozaki pass: probe check + timings, parity tests, cfg4 bench
O=gpurun_out/rp; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
OZ_F32=1 timeout 120 ./tools/test_ozaki_base 3000 1500 0 0 128 > $O/check_rp.log 2>&1; echo "rc $?" >> $O/check_rp.log
for v in base SKIP_MMA; do echo "== mode 3 $v";
  OZ_F32=1 OZ_NOCHECK=1 timeout 120 ./tools/test_ozaki_$v 250000 10000 5 0 128 2>&1 | grep "trans"; done > $O/probe_rp.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "fp32 or config4" -rs > $O/pytest_fp32.log 2>&1; echo "pytest rc $?" >> $O/pytest_fp32.log
timeout 600 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_cfg4.log 2>&1; echo "rc $?" >> $O/bench_cfg4.log
