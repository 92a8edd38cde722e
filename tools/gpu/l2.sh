O=gpurun_out/l2; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k 'regex:rsvd::|oz::' -c 2000 --csv \
  --log-file $O/launches_cfg2.csv python bench.py --config 2 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_launches2.log 2>&1
echo "rc $?"
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:ozaki_pass_kernel<1' -s 2 -c 1 \
  -o $O/cfg3_pass_tn python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_full_tn.log 2>&1; echo "rc $?"
tail -3 $O/ncu_full_tn.log
