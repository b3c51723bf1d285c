timeout 600 python -m pytest tests/test_gpu_checkpoint_eval.py -x -q 2>&1 | tail -25
