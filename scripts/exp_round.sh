mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ffca_loop -c 1 -f -o gpurun_out/r2f_c2 python scripts/run_once.py 2 > gpurun_out/r2f_c2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:point_tile -c 2 -f -o gpurun_out/r2f_points python scripts/points_bench.py c64 > gpurun_out/r2f_points.log 2>&1
