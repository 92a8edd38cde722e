timeout 120 ./tools/test_ozaki_base 3000 1100 5 0 2>&1 | grep -v "^  C\|^  R\|MMA thread\|producer"
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -x --deselect "tests/test_gpu_parity.py::test_rrpca_adaptive_and_large_rank_parity[3000-400-40-60]" > gpurun_out/rows_pytest.log 2>&1; echo pytest rc $?
tail -3 gpurun_out/rows_pytest.log
for c in 2 3 5; do timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/rows_cfg$c.log 2>&1; echo cfg$c rc $?; done
