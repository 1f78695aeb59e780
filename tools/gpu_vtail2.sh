set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "tail" > gpurun_out/vtail_tests2.log 2>&1; echo "rc=$?" >> gpurun_out/vtail_tests2.log
timeout 300 python tools/profile_path.py --what vtailtl > gpurun_out/vtail_tl.log 2>&1
