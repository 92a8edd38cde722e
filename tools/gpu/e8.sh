echo "== probe"; OZ_TIMELINE=1 RSVD_OZ_BK=64 timeout 120 ./tools/test_ozaki_base 10000 5000 20 0 64 2>&1 | grep "trans\|us:"
RSVD_OZ_BK=64 timeout 120 ./tools/test_ozaki_base 20000 4000 10 0 128 2>&1 | grep "trans"
RSVD_OZ_BK=32 timeout 120 ./tools/test_ozaki_base 10000 5000 20 0 64 2>&1 | grep "trans"
for bk in 64 32; do RSVD_OZ_BK=$bk timeout 300 python bench.py --config 2 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/e8_bk${bk}_cfg2.log 2>&1; echo rc $?; done
for bk in 64 32; do RSVD_OZ_BK=$bk timeout 300 python bench.py --config 3 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/e8_bk${bk}_cfg3.log 2>&1; echo rc $?; done
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/e8_pytest.log 2>&1; echo pytest rc $?
tail -3 gpurun_out/e8_pytest.log
