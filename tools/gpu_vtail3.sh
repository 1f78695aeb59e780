set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_abi_layout.py -x -q -k "tail or layout" > gpurun_out/vtail_tests3.log 2>&1; echo "rc=$?" >> gpurun_out/vtail_tests3.log
for kb in 150 80; do
echo "== vec $kb" >> gpurun_out/vtail_time3.log
CPRB_TAIL_VEC_KB=$kb timeout 300 python tools/profile_path.py --what vcycleg --reps 200 >> gpurun_out/vtail_time3.log 2>&1
CPRB_TAIL_VEC_KB=$kb timeout 300 python tools/profile_path.py --what vtailtl > gpurun_out/vtail_tl3_$kb.log 2>&1
CPRB_TAIL_VEC_KB=$kb CPRB_TAIL_NOPERSIST=1 timeout 300 python tools/profile_path.py --what vcycleg --reps 200 >> gpurun_out/vtail_time3.log 2>&1
done
CPRB_TAIL_ROWS=0 timeout 300 python tools/profile_path.py --what vcycleg --reps 200 >> gpurun_out/vtail_time3.log 2>&1
