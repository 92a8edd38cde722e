for v in base NOEPI SKIP_MMA SKIPMMA_NOEPI NO_X_TMA; do echo "== $v"; OZ_TIMELINE=1 timeout 300 ./tools/test_ozaki_$v 40000 4000 5 0 128 2>&1 | grep "trans\|us:\|MMA thread\|producer"; done
