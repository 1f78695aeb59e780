mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/full4_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/full4_pytest.log
timeout 600 python bench.py > gpurun_out/full4_bench.log 2>&1; echo "rc=$?" >> gpurun_out/full4_bench.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/full4_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/full4_smoke.log
tail -n 5 gpurun_out/full4_pytest.log; tail -n 3 gpurun_out/full4_bench.log; tail -n 2 gpurun_out/full4_smoke.log
