# A/B of two builds on a 1D multigrid batch (A = libhwgpu_ab.so via HWG_LIB_PATH)
A=$PWD/paper_2009_08875_b200/libhwgpu_ab.so
for i in 1 2 3; do
  echo "A $(HWG_LIB_PATH=$A python scripts/profile_mg.py --d 1 --J 14 --K 10 --reps 5 2>&1 | tail -1)"
  echo "B $(python scripts/profile_mg.py --d 1 --J 14 --K 10 --reps 5 2>&1 | tail -1)"
done
