# Round-2 final evidence: tests, smoke, bench lines (configs 1-5 + reference arm), ncu launch list,
# per-launch pass traffic (configs 2, 3, 4), ncu --set full of the FP32 row-pair pass.
O=gpurun_out/final; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.log 2>&1
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc $?" >> $O/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; echo "smoke rc $?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_default.log 2>&1; echo "rc $?" >> $O/bench_default.log
for c in 1 2 4 5; do timeout 1200 python bench.py --config $c > $O/bench_cfg$c.log 2>&1; echo "rc $?" >> $O/bench_cfg$c.log; done
timeout 900 python bench.py --impl reference > $O/bench_reference.log 2>&1; echo "rc $?" >> $O/bench_reference.log
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k 'regex:rsvd::|oz::' -c 2000 --csv \
  --log-file $O/launches_cfg3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_launches.log 2>&1
echo "rc $?" >> $O/ncu_launches.log
for c in 3 2 4 5; do
timeout 1200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:ozaki_pass_kernel -c 4 --csv \
  --log-file $O/traffic_cfg$c.csv python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_traffic_cfg$c.log 2>&1
echo "rc $?" >> $O/ncu_traffic_cfg$c.log
done
timeout 300 python tools/prof_fp32.py > $O/prof_fp32_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"ozaki_slice|ozaki_pass_kernel" -s 9 -c 5 \
  -o $O/fp32_rowpair python tools/prof_fp32.py > $O/ncu_fp32.log 2>&1; echo "rc $?" >> $O/ncu_fp32.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"ozaki_pass_kernel<1" -s 2 -c 1 \
  -o $O/cfg3_pass_tn python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_full_tn.log 2>&1; echo "rc $?" >> $O/ncu_full_tn.log
