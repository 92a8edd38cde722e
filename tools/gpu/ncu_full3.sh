timeout 900 ncu --set full --import-source on --clock-control none -k regex:ozaki_slice_rows -c 1 -o gpurun_out/r02_cfg3_slice \
  python bench.py --config 3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full3_slice.log 2>&1
timeout 1500 ncu --set full --import-source on --clock-control none -k 'regex:ozaki_pass_kernel<1' -c 1 -o gpurun_out/r02_cfg3_pass_tn \
  python bench.py --config 3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full3_pass.log 2>&1
echo done >> gpurun_out/ncu_full3_pass.log
