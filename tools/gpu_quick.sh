timeout 600 python tools/gpu_debug.py 2>&1 | tail -12
timeout 300 python tools/stress_admit.py --iters 30 2>&1 | tail -12
timeout 300 python tools/stress_admit.py --iters 30 --mode adversarial 2>&1 | tail -12
