set -x
mkdir -p gpurun_out
./tools/micro/cphase > gpurun_out/cphase.log 2>&1
timeout 600 python tools/debug_ktail.py > gpurun_out/debug_ktail.log 2>&1
