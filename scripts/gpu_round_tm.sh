# Round-2 final pass after the tensor-memory plans: tests, smoke, bench (+ reference arm), launch
# list, and ncu --set full captures of the config-3 (bench) and config-2 loop kernels.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -m gpu -x -q > gpurun_out/r2tm_gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2tm_gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2tm_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/r2tm_bench.json 2> gpurun_out/r2tm_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/r2tm_bench_ref.json 2> gpurun_out/r2tm_bench_ref.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"ffca|slab|point|inv_PH|ll_reduce" -c 400 --csv --log-file gpurun_out/r2tm_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-extra --no-parity > gpurun_out/r2tm_ncu.log 2>&1; echo "launches rc=$?"
[ -n "$NCU_FULL" ] && timeout 900 ncu --set full --clock-control none --import-source on -k regex:ffca_loop -c 1 -f -o gpurun_out/r2tm_c3 python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-extra --no-parity > gpurun_out/r2tm_c3.log 2>&1; echo "c3 rc=$?"
[ -n "$NCU_FULL" ] && timeout 900 ncu --set full --clock-control none --import-source on -k regex:ffca_loop -c 1 -f -o gpurun_out/r2tm_c2 python scripts/run_once.py 2 > gpurun_out/r2tm_c2.log 2>&1; echo "c2 rc=$?"
timeout 300 python scripts/config_sweep.py > gpurun_out/r2tm_config_sweep.log 2>&1; echo "sweep rc=$?"
tail -3 gpurun_out/r2tm_gputest.log
timeout 300 python scripts/pipeline_bench.py > gpurun_out/r2tm_pipeline_bench.json 2> gpurun_out/r2tm_pipeline_bench.err; echo "pipeline rc=$?"
for c in 3 2 4; do CFG=$c timeout 200 python scripts/points_bench.py c64; CFG=$c timeout 200 python scripts/back_bench.py; done > gpurun_out/r2tm_output_kernels.log 2>&1; echo "outputs rc=$?"
