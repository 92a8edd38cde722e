for i in 1 2; do
for v in 0 1; do
  if [ $v = 1 ]; then export RSVD_DEBUG_NO_FALLBACK=1; else unset RSVD_DEBUG_NO_FALLBACK; fi
  for c in 2 3; do timeout 600 python bench.py --config $c --steps 30 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/fb${v}_${i}_cfg$c.log 2>&1; done
done; done
