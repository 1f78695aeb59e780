set -x
mkdir -p gpurun_out
timeout 300 python tools/setup_profile.py > gpurun_out/setup_profile2.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "not slow" > gpurun_out/pytest_fast.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_fast.log
timeout 900 python tools/c4_mix_probe.py > gpurun_out/c4_mix.log 2>&1
