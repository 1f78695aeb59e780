set -x
mkdir -p gpurun_out
K="spe10_shape_c3_against_reference or c4_sequence_reuse"
for i in 1 2 3; do
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "$K" > gpurun_out/r5_default_$i.log 2>&1; echo "rc=$?" >> gpurun_out/r5_default_$i.log
done
timeout 2400 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -x -q -k "$K" > gpurun_out/r5_memcheck.log 2>&1; echo "rc=$?" >> gpurun_out/r5_memcheck.log
