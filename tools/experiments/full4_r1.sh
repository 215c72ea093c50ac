timeout 2400 python -m pytest tests -m gpu -q -x --durations=8 2>&1 | tail -14
