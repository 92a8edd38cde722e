# wide plans (l > 120): new parity tests, then the rsvd / rrpca parity files
O=gpurun_out/wide; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_wide.py -q -x -p no:cacheprovider > $O/pytest_wide.log 2>&1; echo "wide rc $?" >> $O/pytest_wide.log
tail -30 $O/pytest_wide.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "rrpca or tiny or parity_cases" > $O/pytest_rr.log 2>&1; echo "rr rc $?" >> $O/pytest_rr.log
tail -5 $O/pytest_rr.log
