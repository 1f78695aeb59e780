set -x
mkdir -p gpurun_out
K="spe10_shape_c3_against_reference or c4_sequence_reuse"
CPRB_SETUP_SYNC=1 timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "$K" > gpurun_out/r4_sync.log 2>&1; echo "rc=$?" >> gpurun_out/r4_sync.log
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "$K" > gpurun_out/r4_default.log 2>&1; echo "rc=$?" >> gpurun_out/r4_default.log
