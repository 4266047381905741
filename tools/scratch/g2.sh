for v in 0 4; do SP_BCC_TET_VARIANT=$v python tools/prof_eval.py --workload bcc_linear_2x203_fp32 --iters 10; done
for v in 0 4; do SP_BCC_TET_VARIANT=$v python tools/prof_eval.py --workload bcc_linear_2x406_1e9_fp32 --iters 3; done
SP_BCC_TET_VARIANT=0 ncu --set full --clock-control none --import-source on -k regex:bcc_tet -s 1 -c 1 -o gpurun_out/r2c_bcc_linear_v2 python tools/prof_eval.py --workload bcc_linear_2x203_fp32 --iters 2 > /dev/null 2>&1; echo ncu rc $?
