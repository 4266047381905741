python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -x -q -m gpu -k "bcc_linear" 2>&1 | tail -2
for v in 0 3; do SP_BCC_TET_VARIANT=$v python tools/prof_eval.py --workload bcc_linear_2x203_fp32 --iters 10; done
for v in 0 3; do SP_BCC_TET_VARIANT=$v python tools/prof_eval.py --workload bcc_linear_2x406_1e9_fp32 --iters 3; done
python tools/prof_eval.py --workload bcc_linear_2x203_fp64 --iters 10
