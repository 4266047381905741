for w in tricubic_cc256_fp32 bcc_linear_2x203_fp32; do
for ppt in 1 2 4 8; do for kb in 24 40 64 96; do SP_PPT=$ppt SP_TILE_KB=$kb python tools/prof_eval.py --workload $w --iters 5; done; done; done
