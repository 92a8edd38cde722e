# FP32 (3-digit) Ozaki pass probes: full kernel vs no MMA / no A loads / no X loads / no epilogue,
# single-CTA N=128 and the column-pair launch
O=gpurun_out/probe32; mkdir -p $O
for single in 1 0; do for v in base SKIP_MMA NO_A_TMA NO_X_TMA NO_EPI; do
  echo "== single $single $v"
  OZ_F32=1 OZ_NOCHECK=1 RSVD_OZ_SINGLE128=$single timeout 120 ./tools/test_ozaki_$v 250000 10000 5 0 128 2>&1 | grep -v "^  C\|^  R"
done; done > $O/probe32.log 2>&1
OZ_F32=1 timeout 300 ./tools/test_ozaki_base 20000 3000 0 0 > $O/check32.log 2>&1
