# A/B of two builds on the default bench's e2e leg (A = libhwgpu_ab.so via HWG_LIB_PATH)
A=$PWD/paper_2009_08875_b200/libhwgpu_ab.so
for i in 1 2; do
  for v in A B; do
    if [ $v = A ]; then export HWG_LIB_PATH=$A; else unset HWG_LIB_PATH; fi
    python bench.py --steps 2 --warmup 2 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['time_to_solve_s'], d['e2e']['time_to_solve_s'], d['e2e']['value'])"
  done
done
unset HWG_LIB_PATH
