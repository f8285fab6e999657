echo "tests: $(timeout 900 python -m pytest tests/test_gpu_model.py tests/test_gpu_sampling.py tests/test_gpu_disagg.py -q 2>&1 | tail -1)"
timeout 600 python scripts/kprof.py --variant ordinary --warm-rounds 160 --rounds 5 2>&1 | grep -E "phase (d|t)|resid|rope"
