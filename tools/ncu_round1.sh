set -x
NCU=ncu
$NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_solve.csv python tools/profile_path.py --what solve --reps 1 > gpurun_out/ncu_l.log 2>&1
$NCU --set full --clock-control none --import-source on -k regex:k_bsr -s 2 -c 1 -o gpurun_out/prof_bsr python tools/profile_path.py --what spmv --reps 3 > gpurun_out/ncu_b.log 2>&1
$NCU --set full --clock-control none --import-source on -k regex:k_sweep -c 2 -o gpurun_out/prof_sweep python tools/profile_path.py --what vcycle --reps 1 --nograph > gpurun_out/ncu_s.log 2>&1
$NCU --set full --clock-control none --import-source on -k regex:k_wave -c 2 -o gpurun_out/prof_wave python tools/profile_path.py --what bilu --reps 1 --nograph > gpurun_out/ncu_w.log 2>&1
$NCU --set full --clock-control none --import-source on -k regex:k_resid_restrict -c 1 -o gpurun_out/prof_rr python tools/profile_path.py --what vcycle --reps 1 --nograph > gpurun_out/ncu_r.log 2>&1
ls -la gpurun_out
