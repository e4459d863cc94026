mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:point_tile -c 2 -f -o gpurun_out/r2_points2 python scripts/points_bench.py c64 > gpurun_out/ncu_points2.log 2>&1
