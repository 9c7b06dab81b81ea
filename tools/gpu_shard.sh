timeout 900 python -m pytest tests/test_gpu_shard.py -x -q --timeout 300 -k "tight or snapshot or nccl or torch" 2>&1 | tail -15
timeout 600 python bench.py --parallel sharded --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | tail -3
