timeout 900 python -m pytest tests/test_gpu_model.py -x -q 2>&1 | tail -2
for v in 0 1; do for c in 24 8; do echo "== ROPE_VEC=$v CTAS=$c"; SPECTRE_ROPE_VEC=$v SPECTRE_ROPE_CTAS=$c timeout 600 python scripts/kprof.py --variant ordinary --warm-rounds 160 --rounds 3 2>&1 | grep -E "phase (d|t)|rope"; done; done
