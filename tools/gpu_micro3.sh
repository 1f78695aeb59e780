set -x
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/cphase tools/micro/cluster_phase.cu && /tmp/cphase > gpurun_out/cphase2.log 2>&1
