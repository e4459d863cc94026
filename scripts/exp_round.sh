mkdir -p gpurun_out
{
for c in 2 4 2; do python scripts/exp_time.py $c; done
} > gpurun_out/exp15.log 2>&1
timeout 600 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-extra --no-parity > gpurun_out/bench_q.json 2>gpurun_out/bench_q.err
