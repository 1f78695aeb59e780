set -x
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/cphase tools/micro/cluster_phase.cu && /tmp/cphase > gpurun_out/cphase.log 2>&1
timeout 900 python -m pytest tests/test_ktail.py -x -q > gpurun_out/ktail_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ktail_tests.log
timeout 300 python tools/setup_profile.py > gpurun_out/setup_profile.log 2>&1
