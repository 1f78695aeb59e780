mkdir -p gpurun_out
run() { echo "== $G $*" >> gpurun_out/p2.log; env "$@" timeout 240 python tools/repro_rate.py $G >> gpurun_out/p2.log 2>&1; echo "rc=$?" >> gpurun_out/p2.log; }
for G in 60,220,300; do
  run CPRB_STENCIL_MAXCLUS=1 REPS=5
  run CPRB_STENCIL_MAXCLUS=4 REPS=10
  run CPRB_STENCIL_MAXCLUS=8 REPS=10
  run CPRB_STENCIL_MAXCLUS=1000 REPS=10
done
G=120,440,170 run CPRB_STENCIL_MAXCLUS=2 REPS=10
grep -v "^frame" gpurun_out/p2.log | grep -E "^==|OK|rc=|stencil:|Error" 
