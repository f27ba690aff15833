# ncu launch list (per-launch duration + DRAM bytes) of one PCG solve via
# scripts/profile_mg.py --what pcg; args: d J K [domain]
d=$1; J=$2; K=$3; dom=${4:-square}
python scripts/profile_mg.py --d $d --J $J --K $K --what pcg --reps 1 --domain $dom > gpurun_out/profile_pcg_${d}_${J}_${K}.txt 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_pcg_${d}_${J}_${K}.csv python scripts/profile_mg.py --d $d --J $J --K $K --what pcg --reps 1 --domain $dom > gpurun_out/ncu_pcg_${d}_${J}_${K}.log 2>&1
