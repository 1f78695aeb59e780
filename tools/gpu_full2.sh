set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_all2.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_all2.log
timeout 900 python bench.py > gpurun_out/bench2.json 2> gpurun_out/bench2.err
timeout 900 python bench.py --config c4 --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
for tool in memcheck racecheck synccheck; do
timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_c1.py > gpurun_out/sanitize_c1_$tool.log 2>&1
done
timeout 1200 compute-sanitizer --tool memcheck --target-processes all --print-limit 20 python -m pytest tests/test_partition.py -q -x -k "ranks_bitwise_equal and 2-v-0.0 or two_processes_ipc" > gpurun_out/sanitize_slab_memcheck.log 2>&1
