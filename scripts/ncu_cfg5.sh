# ncu evidence for the cfg-5 per-GPU share (mapped L, K = 11): launch list of one
# MG batch at J = 8 (514 rows) and full captures of the n = 2047 DOWN (zero start)
# and UP launches
set -x
python scripts/profile_mg.py --J 8 --K 11 --domain L --reps 1 > gpurun_out/profile_L.txt 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_L_K11.csv python scripts/profile_mg.py --J 8 --K 11 --domain L --reps 1 > gpurun_out/ncu_L.log 2>&1
ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k 'regex:mg2d_reg<\(int\)8, \(int\)256, \(bool\)1, \(bool\)1' -c 1 -o gpurun_out/ncu_L_reg_down_zs python scripts/profile_mg.py --J 8 --K 11 --domain L --reps 1 >> gpurun_out/ncu_L.log 2>&1
ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k 'regex:mg2d_reg<\(int\)8, \(int\)256, \(bool\)0' -c 1 -o gpurun_out/ncu_L_reg_up python scripts/profile_mg.py --J 8 --K 11 --domain L --reps 1 >> gpurun_out/ncu_L.log 2>&1
