set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_device_setup.py tests/test_generator.py tests/test_gpu_parity.py -x -q -k "tail or device_setup or generator or bilu0 or stencil or c1" > gpurun_out/vtail_tests.log 2>&1; echo "rc=$?" >> gpurun_out/vtail_tests.log
for r in 0 100000; do CPRB_TAIL_ROWS=$r timeout 300 python tools/profile_path.py --what vcycleg --reps 200 >> gpurun_out/vtail_time.log 2>&1; CPRB_TAIL_ROWS=$r timeout 300 python tools/profile_path.py --what vcyclecold --reps 50 >> gpurun_out/vtail_time.log 2>&1; done
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_vtail.json 2> gpurun_out/bench_vtail.err
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_all.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_all.log
