set -x
mkdir -p gpurun_out
CPRB_TAIL_ROWS=600 timeout 600 compute-sanitizer --tool memcheck python tools/debug_vtail.py > gpurun_out/dbg_memcheck.log 2>&1
CPRB_TAIL_ROWS=600 CPRB_TAIL_NOPERSIST=1 timeout 300 python tools/debug_vtail.py > gpurun_out/dbg_nopersist.log 2>&1
