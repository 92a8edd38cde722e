for c in 2 3; do timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/slc3_cfg$c.log 2>&1; done
