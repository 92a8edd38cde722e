set -x
O=gpurun_out/final2; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -3 $O/pytest_gpu.log
timeout 900 python tools/stress_determinism.py 20000 > $O/stress_determinism_20000.log 2>&1; echo "stress rc $?"; tail -10 $O/stress_determinism_20000.log
