# k rotation of the TN Ozaki passes: parity, A/B bench (cfg3, cfg4), DRAM traffic of the cfg3 pass
O=gpurun_out/krot; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc $?" >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
for v in 0 1; do
  RSVD_OZ_KROT=$v timeout 600 python bench.py --no-cpu-baseline --no-e2e > $O/bench_cfg3_krot$v.log 2>&1
  python tools/show_bench.py $O/bench_cfg3_krot$v.log 2>/dev/null | head -5 || tail -c 600 $O/bench_cfg3_krot$v.log
done
for v in 1 0; do
  RSVD_OZ_KROT=$v timeout 900 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_cfg4_krot$v.log 2>&1
  python tools/show_bench.py $O/bench_cfg4_krot$v.log 2>/dev/null | head -5 || tail -c 600 $O/bench_cfg4_krot$v.log
done
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:ozaki_pass_kernel -c 4 --csv \
  --log-file $O/traffic_cfg3.csv python bench.py --config 3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_traffic_cfg3.log 2>&1
echo "ncu rc $?"
grep -i "dram__bytes_read\|gpu__time" $O/traffic_cfg3.csv | head -12
