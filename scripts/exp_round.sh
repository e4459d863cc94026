mkdir -p gpurun_out
{
python scripts/points_bench.py c64
FFCA_LIB=build/lib_t3.so python scripts/points_bench.py c64
python scripts/points_bench.py c64
FFCA_LIB=build/lib_t3.so python scripts/points_bench.py c64
} > gpurun_out/exp25.log 2>&1
