# compute-sanitizer on the final round-2 kernels: C1 through every device
# path, and a multi-round persistent stencil case (3 rounds on one cluster)
mkdir -p gpurun_out
S=/usr/local/cuda/bin/compute-sanitizer
timeout 900 $S --tool memcheck python tools/sanitize_c1.py > gpurun_out/r02b_sanitize_c1_memcheck.log 2>&1
timeout 900 $S --tool synccheck python tools/sanitize_c1.py > gpurun_out/r02b_sanitize_c1_synccheck.log 2>&1
CPRB_STENCIL_MAXCLUS=1 REPS=1 timeout 900 $S --tool memcheck python tools/stencil_rounds.py 40,7,33 > gpurun_out/r02b_sanitize_rounds_memcheck.log 2>&1
CPRB_STENCIL_MAXCLUS=1 REPS=1 timeout 900 $S --tool synccheck python tools/stencil_rounds.py 40,7,33 > gpurun_out/r02b_sanitize_rounds_synccheck.log 2>&1
for f in gpurun_out/r02b_sanitize_*.log; do echo "== $f"; grep -E "ERROR SUMMARY|OK|bitwise|Error" $f | tail -4; done
