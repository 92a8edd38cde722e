for v in base EV16 EV4; do echo "== $v"; RSVD_OZ_BK=64 timeout 120 ./tools/test_ozaki_$v 10000 5000 20 0 64 2>&1 | grep "trans"; done
