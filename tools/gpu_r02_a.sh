# Round-2 evidence pass on 1 B200: GPU tests, smoke, bench, launch list, ncu of the BILU stencil kernel.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_solve_r02.csv python tools/profile_path.py --what solve --reps 1 > gpurun_out/ncu_l.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stencil -c 2 -o gpurun_out/r02_stencil python tools/profile_path.py --what bilu --reps 1 > gpurun_out/ncu_w.log 2>&1
ls -la gpurun_out
