mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/exp_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/exp_tests.log
timeout 900 python bench.py --no-cpu-baseline --no-extra > gpurun_out/bench_e2e.json 2> gpurun_out/bench_e2e.err; echo "bench rc=$?" >> gpurun_out/exp_tests.log
