set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm,clocks.sm --format=csv > gpurun_out/r_smi.txt
timeout 600 python bench.py > gpurun_out/r_bench.json 2> gpurun_out/r_bench.err; echo bench rc=$?
timeout 400 python bench.py --impl reference > gpurun_out/r_bench_ref.json 2> gpurun_out/r_bench_ref.err; echo ref rc=$?
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 20 --warmup 3 --headline-only --no-cpu-baseline > gpurun_out/r_torchrun.json 2> gpurun_out/r_torchrun.err; echo torchrun rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r_launches.csv python bench.py --steps 3 --warmup 3 --headline-only --no-cpu-baseline > gpurun_out/r_ncu_launch.log 2>&1; echo launches rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:brick_kernel -s 1 -c 1 -o gpurun_out/r_bcclin python tools/prof_eval.py --workload bcc_linear_2x203_fp32 --iters 2 > gpurun_out/r_bcclin.log 2>&1; echo bcclin rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:brick_kernel_tma -s 1 -c 1 -o gpurun_out/r_tric python tools/prof_eval.py --iters 2 > gpurun_out/r_tric.log 2>&1; echo tric rc=$?
