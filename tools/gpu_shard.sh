timeout 900 python -m pytest tests/test_gpu_shard.py -x -q --timeout 300 2>&1 | tail -5
timeout 600 python bench.py --parallel sharded --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-600
