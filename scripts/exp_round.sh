mkdir -p gpurun_out
{
for r in 1 2 3; do for c in 0 3 2; do python scripts/exp_time.py $c; FFCA_LIB=build/lib_base.so python scripts/exp_time.py $c; done; done
} > gpurun_out/exp17.log 2>&1
python -m pytest tests -m gpu -x -q > gpurun_out/exp_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/exp_tests.log
