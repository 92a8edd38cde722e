timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 2400 > gpurun_out/full2_pytest.log 2>&1; echo pytest rc $?
grep -E "passed|failed|FAILED|Error" gpurun_out/full2_pytest.log | tail -12
