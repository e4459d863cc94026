mkdir -p gpurun_out
{
python scripts/points_bench.py c64
python scripts/points_bench.py c128
} > gpurun_out/exp23.log 2>&1
python -m pytest tests -m gpu -x -q > gpurun_out/exp_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/exp_tests.log
