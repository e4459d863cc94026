mkdir -p gpurun_out
{
python scripts/fixed_probe.py 4 0
python scripts/fixed_probe.py 4 20
python scripts/fixed_probe.py 3 0
python scripts/fixed_probe.py 3 20
python scripts/fixed_probe.py 2 0
python scripts/fixed_probe.py 2 30
} > gpurun_out/fixed.log 2>&1
