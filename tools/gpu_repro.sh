set -x
mkdir -p gpurun_out
timeout 600 compute-sanitizer --tool memcheck --print-limit 10 python tools/repro_c4mix.py 20,30,10 4 0 > gpurun_out/repro_memcheck_small.log 2>&1
CUDA_LAUNCH_BLOCKING=1 timeout 900 python tools/repro_c4mix.py 60,220,85 5 5 > gpurun_out/repro_c3.log 2>&1
timeout 900 compute-sanitizer --tool memcheck --print-limit 10 python tools/repro_c4mix.py 30,110,42 4 0 > gpurun_out/repro_memcheck_mid.log 2>&1
