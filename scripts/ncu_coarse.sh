# full ncu capture of one mg2d_coarse launch below the streamed levels (cfg 2 shape)
ncu --set full --import-source on --clock-control none -k regex:mg2d_coarse -c 1 -o gpurun_out/ncu_coarse python scripts/profile_mg.py --J 8 --K 8 --reps 1 > gpurun_out/ncu_coarse.log 2>&1
