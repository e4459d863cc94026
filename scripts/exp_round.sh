mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/exp_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/exp_tests.log
python scripts/pipeline_bench.py > gpurun_out/r2_pipeline2.log 2>&1
