for v in base KSU64 KSU1K NOEPI; do echo "== $v"; RSVD_OZ_BK=64 timeout 120 ./tools/test_ozaki_$v 10000 5000 20 0 64 2>&1 | grep "trans\|producer\|MMA thread"; done
for v in base KSU1K; do echo "== N=128 $v"; RSVD_OZ_BK=64 timeout 120 ./tools/test_ozaki_$v 20000 4000 10 0 128 2>&1 | grep "trans"; done
