# ncu launch list (per-launch duration + DRAM bytes) of the default bench
# command, bounded to the first 2400 launches (warm-up solve + timed solve)
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 2400 --csv --log-file gpurun_out/launches_bench_cfg4.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
python scripts/launch_summary.py gpurun_out/launches_bench_cfg4.csv > gpurun_out/launch_summary_cfg4.csv
