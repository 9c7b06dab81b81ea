# Round-2 final evidence on the final build: GPU suite, smoke, bench line + reference arm, ncu
# full capture + launch list of the dominant kernel (bound to the sources' src_sha16), the
# sharded pool at N=1 (peer and NCCL) and its phase timeline, the CTA-0 timeline.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest $?
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke $?
tail -1 gpurun_out/smoke.log
CS_SERVER=0 timeout 900 ncu --set full --import-source on --clock-control none -k regex:admit_kernel -s 1600 -c 1 -o gpurun_out/r02_admit_full -f python tools/ncu_admit.py --skip 1600 --n 2 > gpurun_out/ncu_full.log 2>&1; echo ncu_full $?
CS_SERVER=0 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:admit_kernel -c 400 --csv --log-file gpurun_out/r02_admit_launches_dram.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo ncu_list $?
python tools/ncu_summarize.py full gpurun_out/r02_admit_full.ncu-rep gpurun_out/r02_admit_launches_dram.csv > gpurun_out/ncu_admit_summary.json; echo summ $?
cp gpurun_out/ncu_admit_summary.json profiles/ncu_admit_summary.json
timeout 900 python bench.py > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err; echo bench $?
tail -1 gpurun_out/r02_bench.json | cut -c1-300
timeout 900 python bench.py --impl reference > gpurun_out/r02_bench_reference.json 2> gpurun_out/r02_bench_ref.err; echo ref $?
for c in peer nccl; do
timeout 600 python bench.py --parallel sharded --comm $c --steps 20 > gpurun_out/r02_bench_sharded_$c.json 2> gpurun_out/r02_bench_sharded_$c.err; echo sharded_$c $?
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/r02_sharded_launches.csv python bench.py --parallel sharded --no-cpu-baseline --steps 2 --warmup 3 > gpurun_out/ncu_sharded.log 2>&1; echo ncu_sharded $?
timeout 600 python tools/shard_timeline.py > gpurun_out/r02_shard_timeline.txt 2>&1; echo shard_tl $?
timeout 300 python tools/cta0_timeline.py 1600 > gpurun_out/r02_cta0_timeline.txt 2>&1; echo tl $?
