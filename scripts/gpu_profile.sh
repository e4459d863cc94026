# Round-2 profiling pass: launch list of the bench, one ncu --set full capture of the config-3 and
# config-4 loop kernels, and the per-phase probe (build/libffca_probe.so, built in-tree).
mkdir -p gpurun_out
set -x
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"ffca|slab|point|inv_PH|ll_reduce" -c 400 --csv --log-file gpurun_out/r2_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-extra --no-parity > gpurun_out/r2_ncu.log 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ffca_loop -c 1 -f -o gpurun_out/r2_c3 python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-extra --no-parity > gpurun_out/r2_c3.log 2>&1; echo "c3 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ffca_loop -c 1 -f -o gpurun_out/r2_c4 python scripts/run_once.py 4 > gpurun_out/r2_c4.log 2>&1; echo "c4 rc=$?"
timeout 300 python scripts/phase_probe.py 3 > gpurun_out/r2_probe3.log 2>&1; echo "probe3 rc=$?"
timeout 300 python scripts/phase_probe.py 4 > gpurun_out/r2_probe4.log 2>&1; echo "probe4 rc=$?"
