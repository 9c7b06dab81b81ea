timeout 1500 python tools/stress_sweep.py > gpurun_out/r01_stress_sweep.jsonl 2> gpurun_out/stress.err; echo sweep $?
cat gpurun_out/r01_stress_sweep.jsonl
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 2>&1 | tail -1
