set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 600 2>&1 | tail -15
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench $?
tail -1 gpurun_out/bench.json
timeout 600 python tools/bench_timeline.py 2>&1 | tail -12
