timeout 900 python -m pytest tests/test_gpu_multi.py -q -x -k "graph" 2>&1 | tail -3
