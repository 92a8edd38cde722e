for l in 60 120; do
timeout 600 ncu --set full --import-source on --clock-control none -k regex:jacobi_blk -s 2 -c 1 -o gpurun_out/jblk_l$l ./tools/bench_jacobi $l > gpurun_out/jncu_l$l.log 2>&1
done
