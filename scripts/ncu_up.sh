# full ncu capture (with source) of one finest-level UP pass at K = 10 (1026 rows)
ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k 'regex:mg2d_reg<\(int\)8, \(int\)128, \(bool\)0' -c 1 -o gpurun_out/ncu_up python scripts/profile_mg.py --J 9 --K 10 --reps 1 > gpurun_out/ncu_up.log 2>&1
