mkdir -p gpurun_out
{
for r in 1 2; do python scripts/exp_time.py 4; done
} > gpurun_out/exp24.log 2>&1
python -m pytest tests -m gpu -x -q > gpurun_out/exp_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/exp_tests.log
