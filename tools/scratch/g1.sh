set -x
python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "bcc_linear" 2>&1 | tail -3
python -m pytest tests/test_gpu_scale.py -x -q -m gpu -k "bcc_linear" 2>&1 | tail -3
for v in 0 3; do for w in bcc_linear_2x203_fp32 bcc_linear_2x203_fp64; do SP_BCC_TET_VARIANT=$v python tools/prof_eval.py --workload $w --iters 10; done; done
for v in 0 3; do SP_BCC_TET_VARIANT=$v python tools/prof_eval.py --workload bcc_linear_2x406_1e9_fp32 --iters 3; done
