#!/bin/bash
# Build + run the B200 microbenchmarks (under gpurun). Output to gpurun_out/.
set -e
cd "$(dirname "$0")"
mkdir -p ../../gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o /tmp/micro_prox micro_prox.cu
timeout 120 /tmp/micro_prox | tee ../../gpurun_out/micro_prox.log
