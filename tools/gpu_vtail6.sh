set -x
mkdir -p gpurun_out
CPRB_TAIL_ROWS=100000 CPRB_TAIL_MODE=1 CPRB_TAIL_VEC_KB=40 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_vtail -s 2 -c 1 -o gpurun_out/vtail_m1 python tools/profile_path.py --what vcycle --reps 3 --nograph > gpurun_out/ncu_vt1.log 2>&1
CPRB_TAIL_ROWS=100000 CPRB_TAIL_MODE=0 CPRB_TAIL_VEC_KB=40 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_vtail -s 2 -c 1 -o gpurun_out/vtail_m0 python tools/profile_path.py --what vcycle --reps 3 --nograph > gpurun_out/ncu_vt0.log 2>&1
