mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/final_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/final_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/final_smoke.log
timeout 900 python bench.py > gpurun_out/final_bench.log 2>&1; echo "rc=$?" >> gpurun_out/final_bench.log
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/final_bench_ref.log 2>&1; echo "rc=$?" >> gpurun_out/final_bench_ref.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^k_stencil$" -c 2 -o gpurun_out/r02c_stencil python tools/profile_path.py --what bilu --reps 1 > gpurun_out/ncu_w2.log 2>&1
tail -n 3 gpurun_out/final_pytest.log gpurun_out/final_smoke.log; grep -c '"metric"' gpurun_out/final_bench.log gpurun_out/final_bench_ref.log
