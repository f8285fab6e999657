timeout 600 python -m pytest tests/test_gpu_model.py -x -q 2>&1 | tail -2
for v in 2 1; do echo "== pair $v"; SPECTRE_ATTN_WPAIR=$v timeout 300 python scripts/kprof.py --variant ordinary --warm-rounds 160 --rounds 3 2>&1 | grep -v Warn | grep -E "phase draft|k_attn_w<64"; done
