# Scratch driver for one gpurun call (edited per experiment); see scripts/gpu_round.sh for the
# full round (GPU tests, smoke, bench, reference arm, ncu launch list) and scripts/gpu_profile.sh
# for the ncu / probe pass.
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/exp_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/exp_tests.log
