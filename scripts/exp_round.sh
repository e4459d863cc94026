mkdir -p gpurun_out
{
python scripts/exp_time.py 2
FFCA_LIB=build/lib_ck3.so python scripts/exp_time.py 2
FFCA_LIB=build/lib_ck2.so python scripts/exp_time.py 2
python scripts/exp_time.py 2
} > gpurun_out/exp26.log 2>&1
