O=gpurun_out/wide; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_wide.py -q -p no:cacheprovider --durations=12 > $O/pytest_wide.log 2>&1; echo "wide rc $?" >> $O/pytest_wide.log
tail -40 $O/pytest_wide.log
