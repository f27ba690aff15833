# full ncu capture of one bside_fused launch (S-hat B-side) at J = 9, K = 10
ncu --set full --import-source on --clock-control none -k regex:bside_fused -c 1 -o gpurun_out/ncu_bside python scripts/time_schur.py --reps 1 > gpurun_out/ncu_bside.log 2>&1
