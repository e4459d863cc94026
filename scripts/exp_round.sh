mkdir -p gpurun_out
{
python scripts/exp_time.py 2
for v in 2 4; do echo "pfdp $v"; FFCA_LIB=build/lib_pf$v.so FFCA_FORCE_PLAN=1,1,0,256 python scripts/exp_time.py 2; FFCA_LIB=build/lib_pf$v.so python scripts/exp_time.py 2; FFCA_LIB=build/lib_pf$v.so python scripts/exp_time.py 3; done
} > gpurun_out/exp29.log 2>&1
