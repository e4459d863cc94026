mkdir -p gpurun_out
{
DTYPE=c128 python scripts/exp_time.py 3
python scripts/exp_time.py 0
python scripts/exp_time.py 4
} > gpurun_out/exp21.log 2>&1
python -m pytest tests -m gpu -x -q > gpurun_out/exp_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/exp_tests.log
