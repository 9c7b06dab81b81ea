# Round-2 GPU check: full GPU suite, a bench line and the reference arm.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
lscpu | head -20 > gpurun_out/lscpu.txt; nproc >> gpurun_out/lscpu.txt
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 900 --durations=15 > gpurun_out/gputests.log 2>&1; echo tests $?
tail -25 gpurun_out/gputests.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench $?
tail -1 gpurun_out/bench.json
