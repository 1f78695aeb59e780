set -x
mkdir -p gpurun_out
CPRB_TAIL_ROWS=600 timeout 600 compute-sanitizer --tool memcheck python tools/debug_vtail.py > gpurun_out/dbg_memcheck2.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "tail" > gpurun_out/vtail_tests5.log 2>&1; echo "rc=$?" >> gpurun_out/vtail_tests5.log
for mode in 1 0; do for kb in 150 40 20; do
echo "== mode $mode vec $kb" >> gpurun_out/vtail_time5.log
CPRB_TAIL_MODE=$mode CPRB_TAIL_VEC_KB=$kb timeout 300 python tools/profile_path.py --what vcycleg --reps 200 >> gpurun_out/vtail_time5.log 2>&1
CPRB_TAIL_MODE=$mode CPRB_TAIL_VEC_KB=$kb timeout 300 python tools/profile_path.py --what vtailtl > gpurun_out/vtail_tl5_${mode}_$kb.log 2>&1
done; done
CPRB_TAIL_ROWS=0 timeout 300 python tools/profile_path.py --what vcycleg --reps 200 >> gpurun_out/vtail_time5.log 2>&1
