# A/B of the Ozaki L2 prefetch distance on one box (cfg2, cfg3)
nproc; free -g | head -2
for pf in 0 1 2 4; do
  RSVD_OZ_PF=$pf timeout 300 python bench.py --config 2 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/pf${pf}_cfg2.log 2>&1; echo pf $pf rc $?
done
for pf in 0 2; do
  RSVD_OZ_PF=$pf timeout 600 python bench.py --config 3 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/pf${pf}_cfg3.log 2>&1; echo pf $pf cfg3 rc $?
done
