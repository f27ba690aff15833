# full ncu capture of one 1D multigrid batch (mg1d_reg<10, 8>) at J = 14, K = 10
python scripts/profile_mg.py --d 1 --J 14 --K 10 --reps 1 > gpurun_out/profile_mg1d.txt 2>&1
ncu --set full --import-source on --clock-control none -k regex:mg1d_reg -c 1 -o gpurun_out/ncu_mg1d python scripts/profile_mg.py --d 1 --J 14 --K 10 --reps 1 > gpurun_out/ncu_mg1d.log 2>&1
