# Round-2 final evidence on 1 B200: launch list of one C3 solve (cold,
# serialised), ncu --set full of the stencil L/U kernels, the V-cycle
# critical-path log and the stencil per-plane timeline.
set -x
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_solve_r02b.csv python tools/profile_path.py --what solve --reps 1 > gpurun_out/ncu_l.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stencil -c 2 -o gpurun_out/r02b_stencil python tools/profile_path.py --what bilu --reps 1 > gpurun_out/ncu_w.log 2>&1
AMGTL_OUT=gpurun_out/amgtl_r02b.npy timeout 300 python tools/profile_path.py --what amgtl > gpurun_out/amgtl_r02b.log 2>&1
ALL=1 timeout 300 python tools/stencil_tl.py 60,220,85 > gpurun_out/stencil_tl_r02b.log 2>&1
ls -la gpurun_out | tail -20
