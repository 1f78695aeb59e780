mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_stencil.py tests/test_device_setup.py -m gpu -x -q > gpurun_out/st1_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/st1_pytest.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/st1_bench.log 2>&1; echo "rc=$?" >> gpurun_out/st1_bench.log
tail -n 3 gpurun_out/st1_pytest.log
