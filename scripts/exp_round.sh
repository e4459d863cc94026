mkdir -p gpurun_out
{
for c in 2 3 4 0; do python scripts/exp_time.py $c; done
} > gpurun_out/exp14.log 2>&1
python -m pytest tests -m gpu -x -q > gpurun_out/exp_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/exp_tests.log
