set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "rebuild_mix" > gpurun_out/repro_mix_alone.log 2>&1; echo "rc=$?" >> gpurun_out/repro_mix_alone.log
nvidia-smi --query-gpu=memory.used,memory.total --format=csv >> gpurun_out/repro_mix_alone.log
timeout 2400 python -m pytest tests/test_gpu_parity.py tests/test_partition.py -x -q -k "c4 or c5 or spe10" > gpurun_out/repro_mix_seq.log 2>&1; echo "rc=$?" >> gpurun_out/repro_mix_seq.log
