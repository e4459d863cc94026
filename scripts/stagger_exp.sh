mkdir -p gpurun_out
for s in 0 1500 3000 6000 0; do echo "stagger $s"; FFCA_STAGGER=$s python scripts/config_sweep.py 3; done > gpurun_out/stagger.log 2>&1
