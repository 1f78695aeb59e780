set -x
mkdir -p gpurun_out
K="spe10_shape_c3_against_reference or c4_sequence_reuse"
CUDA_LAUNCH_BLOCKING=1 timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "$K" > gpurun_out/r3_blocking.log 2>&1; echo "rc=$?" >> gpurun_out/r3_blocking.log
CPRB_DEVICE_SETUP=0 timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "$K" > gpurun_out/r3_hostsetup.log 2>&1; echo "rc=$?" >> gpurun_out/r3_hostsetup.log
CPRB_SETUP_THREADS=1 timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "$K" > gpurun_out/r3_serial.log 2>&1; echo "rc=$?" >> gpurun_out/r3_serial.log
CPRB_STENCIL=0 timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "$K" > gpurun_out/r3_nostencil.log 2>&1; echo "rc=$?" >> gpurun_out/r3_nostencil.log
