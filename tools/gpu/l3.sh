O=gpurun_out/l3; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:chol_blk_kernel -s 20 -c 1 \
  -o $O/chol_cfg2 python bench.py --config 2 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_chol.log 2>&1; echo "rc $?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ozaki_pass_kernel -s 3 -c 1 \
  -o $O/cfg3_pass_tn python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_full_tn.log 2>&1; echo "rc $?"
tail -2 $O/ncu_chol.log $O/ncu_full_tn.log
