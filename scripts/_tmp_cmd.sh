timeout 600 python -m pytest tests/test_gpu_sampling.py -x -q 2>&1 | tail -25
timeout 600 python -m pytest tests/test_gpu_model.py -x -q 2>&1 | tail -2
