# Ozaki pass probes: full kernel vs no MMA / no A loads / no X loads, BK 32 and 64
for bk in 64 32; do for v in base SKIP_MMA NO_A_TMA NO_X_TMA; do
  echo "== bk $bk $v"; RSVD_OZ_BK=$bk timeout 120 ./tools/test_ozaki_$v 10000 5000 20 0 64 2>&1 | grep -v "^  C\|^  R"
done; done
