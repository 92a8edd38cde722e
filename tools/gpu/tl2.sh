OZ_TIMELINE=1 timeout 120 ./tools/test_ozaki_base 10000 5000 20 0 64 2>&1 | grep "trans\|us:"
