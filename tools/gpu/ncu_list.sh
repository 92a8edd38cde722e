C=${1:-2}
timeout 600 python bench.py --config $C --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/nl_cfg$C.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k 'regex:rsvd::|oz::' -c ${2:-3000} --csv --log-file gpurun_out/launches_cfg$C.csv \
  python bench.py --config $C --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_cfg$C.log 2>&1
echo rc $? >> gpurun_out/ncu_cfg$C.log
