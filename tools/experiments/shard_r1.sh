timeout 900 python -m pytest tests/test_gpu_multi.py -q -x -s -k "sharded" 2>&1 | grep -E "ok|FAIL|passed|failed|update" | tail -8
