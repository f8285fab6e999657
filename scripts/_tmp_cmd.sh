for v in 0 1; do echo "== GU_SK=$v"; SPECTRE_GU_SK=$v timeout 600 python scripts/kprof.py --variant ordinary --warm-rounds 160 --rounds 3 2>&1 | grep -E "phase|<2, 64, 0>"; done
