set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_device_setup.py tests/test_generator.py -x -q > gpurun_out/devsetup_tests.log 2>&1; echo "rc=$?" >> gpurun_out/devsetup_tests.log
timeout 300 python tools/setup_profile.py > gpurun_out/setup_profile3.log 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_all.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_all.log
