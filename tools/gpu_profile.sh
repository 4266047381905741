#!/bin/bash
# usage (on the GPU box): tools/gpu_profile.sh WORKLOAD TAG [POINTS] [KERNEL_REGEX]
# plain run first (must exit 0), then one ncu --set full capture of the eval kernel.
W=${1:-tricubic_cc256_fp32}; TAG=${2:-prof}; P=${3:-20000000}; K=${4:-"eval_kernel|brick_kernel"}
mkdir -p gpurun_out
python tools/prof_eval.py --workload $W --points $P --iters 2 > gpurun_out/${TAG}_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"$K" -s 2 -c 1 \
    -o gpurun_out/${TAG} python tools/prof_eval.py --workload $W --points $P --iters 2 > gpurun_out/${TAG}_ncu.log 2>&1
echo "profile rc=$?"
