O=gpurun_out/san; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
compute-sanitizer --version > $O/version.log 2>&1
for tool in memcheck racecheck synccheck; do
  timeout 600 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 python tools/sanitize.py > $O/sanitize_$tool.log 2>&1; echo "$tool rc $?" >> $O/sanitize_$tool.log
  tail -6 $O/sanitize_$tool.log
done
