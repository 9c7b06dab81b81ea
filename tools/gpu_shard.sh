timeout 900 python -m pytest tests/test_gpu_shard.py -x -q --timeout 300 2>&1 | tail -30
