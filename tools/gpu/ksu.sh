for v in base K64 K128; do
  echo "== $v" >> gpurun_out/ksu2.log
  timeout 300 ./tools/test_ozaki_$v 10000 5000 20 0 64 >> gpurun_out/ksu2.log 2>&1
  timeout 600 ./tools/test_ozaki_$v 100000 4000 10 0 128 >> gpurun_out/ksu2.log 2>&1
done
