set -x
mkdir -p gpurun_out
for kb in 20 40; do
CPRB_TAIL_ROWS=100000 CPRB_TAIL_MODE=0 CPRB_TAIL_VEC_KB=$kb timeout 300 python tools/profile_path.py --what vtailtl > gpurun_out/vtail_tl7_$kb.log 2>&1
done
