timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/jab_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/jab_pytest.log
for i in 1 2; do
  for v in blk cyc; do
    if [ $v = cyc ]; then export RSVD_JACOBI_CYCLIC=1; else unset RSVD_JACOBI_CYCLIC; fi
    timeout 600 python bench.py --config 2 --steps 30 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/jab_${v}_$i.log 2>&1
    timeout 600 python bench.py --config 1 --steps 30 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/jab1_${v}_$i.log 2>&1
  done
done
