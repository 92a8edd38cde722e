# Final build: ncu launch list of the default bench command and a full capture of the
# config-3 A.X (NN) pass, the kernel bench.py's roofline names.
set -x
O=gpurun_out/final2; mkdir -p $O
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_pre.log 2>&1; echo "bench rc $?"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k 'regex:rsvd::|oz::' -c 2000 --csv \
  --log-file $O/launches_cfg3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_launches.log 2>&1
echo "rc $?" >> $O/ncu_launches.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"ozaki_pass_kernel<0" -s 2 -c 1 \
  -o $O/cfg3_pass_nn python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_full_nn.log 2>&1; echo "rc $?" >> $O/ncu_full_nn.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"jacobi_blk_kernel" -s 2 -c 1 \
  -o $O/cfg3_jacobi python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_full_jac.log 2>&1; echo "rc $?" >> $O/ncu_full_jac.log
ls -la $O
