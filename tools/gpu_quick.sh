timeout 1200 python -m pytest tests -m gpu -x -q --timeout 600 2>&1 | tail -3
timeout 600 python tools/gpu_debug.py 2>&1 | tail -1
timeout 600 python tools/bench_timeline.py 2>&1 | tail -6
timeout 600 python bench.py --no-cpu-baseline 2>&1 | tail -1
