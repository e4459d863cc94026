mkdir -p gpurun_out
{
python scripts/exp_time.py 2
for p in 1,4,1,256 1,8,1,256 1,4,1,128 1,16,1,128 1,16,1,64; do echo "plan $p"; FFCA_FORCE_PLAN=$p python scripts/exp_time.py 2; done
} > gpurun_out/exp22.log 2>&1
