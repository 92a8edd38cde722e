# FP32 Ozaki: ncu --set full of the slicer and the NN / TN passes (second rsvd call)
O=gpurun_out/prof32; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 300 python tools/prof_fp32.py > $O/prof_plain.log 2>&1; echo "rc $?" >> $O/prof_plain.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"ozaki_slice_rows|ozaki_pass_kernel" -s 5 -c 3 \
  -o $O/fp32 python tools/prof_fp32.py > $O/ncu.log 2>&1; echo "rc $?" >> $O/ncu.log
