# Round-2 evidence: ncu captures of the dominant kernel (launch mode, see tools/ncu_summarize.py),
# the per-kernel sweep, the CTA-0 timeline, the stress sweeps and one full bench line + reference arm.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
CS_SERVER=0 timeout 900 ncu --set full --import-source on --clock-control none -k regex:admit_kernel -s 1600 -c 1 -o gpurun_out/r02_admit_full python tools/ncu_admit.py --skip 1600 --n 2 > gpurun_out/ncu_full.log 2>&1; echo ncu_full $?
CS_SERVER=0 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:admit_kernel -c 400 --csv --log-file gpurun_out/r02_admit_launches_dram.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo ncu_list $?
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02_kernels.csv python tools/kernel_sweep.py > gpurun_out/kernel_sweep.out 2>&1; echo ncu_kernels $?
timeout 300 python tools/kernel_sweep.py > gpurun_out/kernel_sweep_host.out 2>&1; echo sweep_host $?
timeout 300 python tools/cta0_timeline.py 1600 > gpurun_out/r02_cta0_timeline.txt 2>&1; echo tl $?
timeout 1200 python tools/stress_sweep.py --pools 1048576,4194304,16777216,67108864 --modes realistic,adversarial --agents 256 > gpurun_out/r02_stress_sweep.jsonl 2> gpurun_out/stress.err; echo stress $?
timeout 1200 python tools/stress_sweep.py --pools 1048576,16777216 --modes realistic --agents 8,32,128,512,1024 > gpurun_out/r02_stress_agents.jsonl 2> gpurun_out/stress_a.err; echo stress_a $?
timeout 900 python bench.py > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err; echo bench $?
tail -1 gpurun_out/r02_bench.json
timeout 900 python bench.py --impl reference > gpurun_out/r02_bench_reference.json 2> gpurun_out/r02_bench_ref.err; echo ref $?
tail -1 gpurun_out/r02_bench_reference.json
lscpu | head -20 > gpurun_out/lscpu.txt; nproc >> gpurun_out/lscpu.txt
