# A/B of two builds on cfg 2 (A = libhwgpu_ab.so via HWG_LIB_PATH)
A=$PWD/paper_2009_08875_b200/libhwgpu_ab.so
for i in 1 2; do
  for v in A B; do
    if [ $v = A ]; then export HWG_LIB_PATH=$A; else unset HWG_LIB_PATH; fi
    python bench.py --config 2 --steps 5 --warmup 2 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v cfg2', d['time_to_solve_s'], d['config']['iterations_per_solve'], d['kernel_classes_ms']['mg2d_coarse'])"
  done
done
unset HWG_LIB_PATH
