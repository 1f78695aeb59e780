# ncu evidence for the committed kernels (run under gpurun on 1 B200):
#   launch list of one C3 solve + full captures of the dominant kernels.
set -x
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_solve_final.csv python tools/profile_path.py --what solve --reps 1 > gpurun_out/ncu_l.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_wave -c 2 -o gpurun_out/final_wave python tools/profile_path.py --what bilu --reps 1 > gpurun_out/ncu_w.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_bsr -s 2 -c 1 -o gpurun_out/final_bsr python tools/profile_path.py --what spmv --reps 3 > gpurun_out/ncu_b.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_sweep -c 2 -o gpurun_out/final_sweep python tools/profile_path.py --what vcycle --reps 1 --nograph > gpurun_out/ncu_s.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_resid_restrict -c 1 -o gpurun_out/final_rr python tools/profile_path.py --what vcycle --reps 1 --nograph > gpurun_out/ncu_r.log 2>&1
ls -la gpurun_out
