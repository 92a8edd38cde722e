timeout 1500 ncu --set full --import-source on --clock-control none -k regex:ozaki_pass_kernel -s 1 -c 1 -o gpurun_out/r02_cfg3_pass_tn \
  python bench.py --config 3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full3_pass.log 2>&1
echo "rc $?" >> gpurun_out/ncu_full3_pass.log
