#!/bin/bash
# Round-end evidence on the GPU box: bench line (ours + reference arm), a torchrun launch,
# the ncu launch list of the headline run, and ncu --set full captures of the hot kernels.
# usage (via gpurun): bash tools/refresh_artifacts.sh [TAG] > gpurun_out/r_refresh.log 2>&1
# Each capture runs only after the same command exited 0 without ncu.
set -x
TAG=${1:-r}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm,clocks.sm --format=csv > gpurun_out/${TAG}_smi.txt
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo bench rc=$?
timeout 400 python bench.py --impl reference > gpurun_out/${TAG}_bench_ref.json 2> gpurun_out/${TAG}_bench_ref.err; echo ref rc=$?
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 20 --warmup 3 --headline-only --no-cpu-baseline > gpurun_out/${TAG}_torchrun.json 2> gpurun_out/${TAG}_torchrun.err; echo torchrun rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 3 --warmup 3 --headline-only --no-cpu-baseline > gpurun_out/${TAG}_ncu_launch.log 2>&1; echo launches rc=$?
for w in tricubic_cc256_fp32:brick_kernel_tma:0 bcc_linear_2x203_fp32:brick_kernel:0 bcc_quintic_2x203_fp32:brick_kernel:0 fcc6_4x161_fp32:brick_kernel:0 zp3_cc256_fp32:brick_kernel:0 c5_fcc_voronoi1_4x322_1e9_fp32:brick_kernel:0 c5_bcc_voronoi1_2x406_1e9_fp32:brick_kernel:0; do
  IFS=: read -r wl k pts <<< "$w"
  extra=""; [ "$pts" != 0 ] && extra="--points $pts"
  timeout 300 python tools/prof_eval.py --workload $wl --iters 2 $extra > gpurun_out/${TAG}_${wl}_plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 -o gpurun_out/${TAG}_$wl python tools/prof_eval.py --workload $wl --iters 2 $extra > gpurun_out/${TAG}_$wl.log 2>&1; echo $wl rc=$?
  # summaries on the box (gpurun brings back <= 64 MiB): keep the report of the headline only
  { python tools/ncu_summary.py gpurun_out/${TAG}_$wl.ncu-rep; echo; echo '## per-source-line (tools/ncu_lines.py)'; echo '```'; python tools/ncu_lines.py gpurun_out/${TAG}_$wl.ncu-rep 30; echo '```'; } > gpurun_out/${TAG}_${wl}_ncu.md 2>&1
  [ "$wl" = tricubic_cc256_fp32 ] || rm -f gpurun_out/${TAG}_$wl.ncu-rep
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:prefilter -s 3 -c 1 -o gpurun_out/${TAG}_prefilter_tma python tools/prof_prefilter.py 1023 > gpurun_out/${TAG}_prefilter_tma.log 2>&1; echo prefilter rc=$?
python tools/ncu_summary.py gpurun_out/${TAG}_prefilter_tma.ncu-rep > gpurun_out/${TAG}_prefilter_tma_ncu.md 2>&1; rm -f gpurun_out/${TAG}_prefilter_tma.ncu-rep
