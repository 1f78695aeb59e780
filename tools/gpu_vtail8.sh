set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "tail" > gpurun_out/vtail_tests8.log 2>&1; echo "rc=$?" >> gpurun_out/vtail_tests8.log
for mode in 0 1; do for kb in 20 40 80 150; do
echo "== mode $mode vec $kb" >> gpurun_out/vtail_time8.log
CPRB_TAIL_ROWS=100000 CPRB_TAIL_MODE=$mode CPRB_TAIL_VEC_KB=$kb timeout 300 python tools/profile_path.py --what vcycleg --reps 200 >> gpurun_out/vtail_time8.log 2>&1
done; done
CPRB_TAIL_ROWS=100000 CPRB_TAIL_MODE=0 CPRB_TAIL_VEC_KB=40 timeout 300 python tools/profile_path.py --what vtailtl > gpurun_out/vtail_tl8.log 2>&1
CPRB_TAIL_ROWS=0 timeout 300 python tools/profile_path.py --what vcycleg --reps 200 >> gpurun_out/vtail_time8.log 2>&1
