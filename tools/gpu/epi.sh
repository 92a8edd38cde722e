for v in base NOEPI SKIP_MMA; do echo "== $v"; RSVD_OZ_BK=64 timeout 120 ./tools/test_ozaki_$v 10000 5000 20 0 64 2>&1 | grep "trans\|producer\|MMA thread"; done
for bk in 64 32; do RSVD_OZ_BK=$bk timeout 300 python bench.py --config 2 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/epi_bk${bk}_cfg2.log 2>&1; echo rc $?; done
for bk in 64 32; do RSVD_OZ_BK=$bk timeout 300 python bench.py --config 3 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/epi_bk${bk}_cfg3.log 2>&1; echo rc $?; done
timeout 600 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/epi_cfg4.log 2>&1; echo rc $?
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "ozaki or config1 or config2 or parity_cases or heterogeneous or tiny or rpca_parity or rqb or fp32" > gpurun_out/epi_pytest.log 2>&1; echo pytest rc $?
tail -3 gpurun_out/epi_pytest.log
