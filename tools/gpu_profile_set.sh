#!/bin/bash
# usage (on the GPU box): tools/gpu_profile_set.sh TAG:WORKLOAD:POINTS:KREGEX ...
# For each item: a plain run first (must exit 0), then one ncu --set full capture of the
# evaluation kernel (the 3rd launch matching KREGEX).
mkdir -p gpurun_out
for item in "$@"; do
  IFS=: read -r TAG W P K <<< "$item"
  python tools/prof_eval.py --workload $W --points $P --iters 2 > gpurun_out/${TAG}_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"$K" -s 2 -c 1 \
      -o gpurun_out/${TAG} python tools/prof_eval.py --workload $W --points $P --iters 2 > gpurun_out/${TAG}_ncu.log 2>&1
  echo "$TAG profile rc=$?"
done
