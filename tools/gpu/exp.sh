for i in 1 2; do for v in 0 1 2 3; do
  export RSVD_TSQR_EXP=$v
  timeout 600 python bench.py --config 2 --steps 30 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/exp${v}_$i.log 2>&1
done; done
