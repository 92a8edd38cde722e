for v in base NOEPI; do echo "== $v"; OZ_TIMELINE=1 timeout 300 ./tools/test_ozaki_$v 40000 4000 5 0 128 2>&1 | grep "trans\|MMA thread\|producer"; done
echo "== N64"; timeout 300 ./tools/test_ozaki_base 10000 5000 20 0 64 2>&1 | grep "trans\|MMA thread"
for c in 2 3; do timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/inc_cfg$c.log 2>&1; echo cfg$c rc $?; done
