# K-cycle tail: bitwise tests, then C3 K solve timings over tail thresholds / CTA sizes.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_ktail.py -x -q > gpurun_out/ktail_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ktail_tests.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "kcycle or c1_against or k0 or kd" > gpurun_out/ktail_parity.log 2>&1; echo "rc=$?" >> gpurun_out/ktail_parity.log
for cfg in "40000 1024" "40000 512" "20000 1024" "10000 1024" "80000 1024"; do
  set -- $cfg
  echo "== rows=$1 threads=$2" >> gpurun_out/ktail_c3.log
  CPRB_KTAIL_ROWS=$1 CPRB_KTAIL_THREADS=$2 timeout 600 python tools/kcycle_c3.py >> gpurun_out/ktail_c3.log 2>&1
done
