set -x
O=gpurun_out/final2; mkdir -p $O
timeout 900 python tools/stress_determinism.py 1000 > $O/stress_determinism.log 2>&1; echo "stress rc $?"; tail -12 $O/stress_determinism.log
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:ozaki_pass_kernel<\(bool\)0' -s 2 -c 1 \
  -o $O/cfg3_pass_nn python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_full_nn.log 2>&1; echo "ncu rc $?"
ls -la $O | grep ncu-rep
