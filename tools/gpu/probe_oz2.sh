# Ozaki pass probes (BK 64): stream vs full kernel, with/without epilogue and PDL; tma_stream reference
for v in base SKIP_MMA SKIPMMA_NOEPI NOEPI; do for pdl in 1 0; do
  echo "== $v pdl $pdl"; RSVD_PDL=$pdl RSVD_OZ_BK=64 timeout 120 ./tools/test_ozaki_$v 10000 5000 20 0 64 2>&1 | grep "trans\|producer\|MMA thread"
done; done
echo "== tma_stream"; timeout 120 ./tools/tma_stream 10000 40 2>&1
