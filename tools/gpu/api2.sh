timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/api2_pytest.log 2>&1; echo pytest rc $?
grep -E "passed|failed|FAILED|Error" gpurun_out/api2_pytest.log | tail -20
