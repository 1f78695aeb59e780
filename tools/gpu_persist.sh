set -x
mkdir -p gpurun_out
for g in 120,440,170 60,220,300 100,100,200 120,440,40; do
  REPS=20 timeout 300 python tools/repro_rate.py $g > gpurun_out/persist_$g.log 2>&1; echo "rc=$?" >> gpurun_out/persist_$g.log
done
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/persist_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/persist_pytest.log
tail -3 gpurun_out/persist_*.log
