set -x
O=gpurun_out/final3; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -2 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc $?"
timeout 900 python bench.py > $O/bench_default.log 2>&1; echo "bench rc $?"; tail -1 $O/bench_default.log | cut -c1-400
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_reference.log 2>&1; echo "ref rc $?"; tail -1 $O/bench_reference.log | cut -c1-300
for c in 4 5; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_cfg$c.log 2>&1; echo "bench$c rc $?"; tail -1 $O/bench_cfg$c.log | cut -c1-200; done
