PYTHONPATH=. timeout 600 python tools/dbg_ranks.py > gpurun_out/dbg_ranks.log 2>&1; cat gpurun_out/dbg_ranks.log
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/full_pytest.log 2>&1; echo pytest rc $?
grep -E "passed|failed|FAILED" gpurun_out/full_pytest.log | tail -8
