for c in 3 2 1; do timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/l2h_cfg$c.log 2>&1; done
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:ozaki_pass -c 4 --csv \
  --log-file gpurun_out/l2h_traffic_cfg3.csv python bench.py --config 3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/l2h_ncu.log 2>&1
echo rc $? >> gpurun_out/l2h_ncu.log
