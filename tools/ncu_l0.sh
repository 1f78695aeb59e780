# ncu --set full of the level-0 sweep colours and residual+restriction (cold L2)
set -x
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep -c 4 -o gpurun_out/r02_sweep python tools/profile_path.py --what vcycle --reps 1 --nograph > gpurun_out/ncu_sweep.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_resid_restrict -c 1 -o gpurun_out/r02_rr python tools/profile_path.py --what vcycle --reps 1 --nograph > gpurun_out/ncu_rr.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_bsr -s 2 -c 1 -o gpurun_out/r02_bsr python tools/profile_path.py --what spmv --reps 3 > gpurun_out/ncu_bsr.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:"k_sweep|k_resid|k_prolong" -c 40 python tools/profile_path.py --what vcycle --reps 1 --nograph > gpurun_out/ncu_l0_list.csv 2>&1
