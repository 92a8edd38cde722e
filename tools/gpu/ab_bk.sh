# A/B of the Ozaki unit size (k per unit) on one box, plus the pass parity tests
for bk in 32 64; do
  RSVD_OZ_BK=$bk timeout 300 python bench.py --config 2 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bk${bk}_cfg2.log 2>&1; echo bk $bk rc $?
  RSVD_OZ_BK=$bk timeout 600 python bench.py --config 3 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bk${bk}_cfg3.log 2>&1; echo bk $bk cfg3 rc $?
done
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "ozaki or config1 or config2 or parity_cases or heterogeneous or tiny or rpca_parity or rqb" > gpurun_out/bk_pytest.log 2>&1; echo pytest rc $?
tail -3 gpurun_out/bk_pytest.log
