mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_stencil.py -m gpu -x -q > gpurun_out/full5_stencil.log 2>&1; echo "rc=$?" >> gpurun_out/full5_stencil.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/full5_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/full5_pytest.log
timeout 600 python bench.py > gpurun_out/full5_bench.log 2>&1; echo "rc=$?" >> gpurun_out/full5_bench.log
for G in 120,440,170 60,220,300; do REPS=10 timeout 300 python tools/repro_rate.py $G >> gpurun_out/full5_rate.log 2>&1; echo "rc=$?" >> gpurun_out/full5_rate.log; done
tail -n 3 gpurun_out/full5_stencil.log gpurun_out/full5_pytest.log; grep -E "OK|rc=" gpurun_out/full5_rate.log
