timeout 1500 python -m pytest tests -m gpu -x -q --timeout 300 2>&1 | tail -3
timeout 600 python bench.py --no-cpu-baseline 2>&1 | tail -1 | cut -c1-1500
