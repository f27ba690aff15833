# A/B of two builds: paper_2009_08875_b200/libhwgpu_ab.so (A, via HWG_LIB_PATH) vs
# the in-tree libhwgpu.so (B); MG batch at K = 10 and the default bench (cfg 4)
A=$PWD/paper_2009_08875_b200/libhwgpu_ab.so
for i in 1 2; do
  echo "A mg $(HWG_LIB_PATH=$A python scripts/profile_mg.py --J 9 --K 10 --reps 5 2>&1 | tail -1)"
  echo "B mg $(python scripts/profile_mg.py --J 9 --K 10 --reps 5 2>&1 | tail -1)"
done
for i in 1 2; do
  for v in A B; do
    if [ $v = A ]; then export HWG_LIB_PATH=$A; else unset HWG_LIB_PATH; fi
    python bench.py --steps 2 --warmup 2 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v cfg4', d['time_to_solve_s'], d['config']['iterations_per_solve'], d['roofline']['frac'])"
  done
done
unset HWG_LIB_PATH
