for i in 1 2; do python tools/prof_eval.py --workload bcc_linear_2x203_fp32 --iters 10; done
python tools/prof_eval.py --workload bcc_linear_2x406_1e9_fp32 --iters 3
