#!/bin/bash
# Round-end evidence on the GPU box: bench line (ours + reference arm), a torchrun launch,
# the ncu launch list of the headline run, and ncu --set full captures of the hot kernels.
# usage (via gpurun): bash tools/refresh_artifacts.sh > gpurun_out/r_refresh.log 2>&1
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm,clocks.sm --format=csv > gpurun_out/r_smi.txt
timeout 900 python bench.py > gpurun_out/r_bench.json 2> gpurun_out/r_bench.err; echo bench rc=$?
timeout 400 python bench.py --impl reference > gpurun_out/r_bench_ref.json 2> gpurun_out/r_bench_ref.err; echo ref rc=$?
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 20 --warmup 3 --headline-only --no-cpu-baseline > gpurun_out/r_torchrun.json 2> gpurun_out/r_torchrun.err; echo torchrun rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r_launches.csv python bench.py --steps 3 --warmup 3 --headline-only --no-cpu-baseline > gpurun_out/r_ncu_launch.log 2>&1; echo launches rc=$?
for w in tricubic_cc256_fp32:brick_kernel_tma bcc_linear_2x203_fp32:brick_kernel bcc_quintic_2x203_fp32:brick_kernel fcc6_4x161_fp32:brick_kernel zp3_cc256_fp32:brick_kernel; do
  wl=${w%%:*}; k=${w##*:}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 -o gpurun_out/r_$wl python tools/prof_eval.py --workload $wl --iters 2 > gpurun_out/r_$wl.log 2>&1; echo $wl rc=$?
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:prefilter -s 3 -c 1 -o gpurun_out/r_prefilter_tma python tools/prof_prefilter.py 1023 > gpurun_out/r_prefilter_tma.log 2>&1; echo prefilter rc=$?
