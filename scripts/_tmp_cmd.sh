timeout 600 python -m pytest tests/test_gpu_gemm.py -x -q 2>&1 | tail -1
SPECTRE_GEMM_KSUB=2 timeout 600 python -m pytest tests/test_gpu_gemm.py -x -q 2>&1 | tail -1
for ks in 0 2; do echo "== engine ksub $ks"; SPECTRE_GEMM_KSUB=$ks timeout 600 python scripts/kprof.py --variant ordinary --warm-rounds 160 --rounds 5 2>&1 | grep -E "phase (d|t)|swapab<1"; done
