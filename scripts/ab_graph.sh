# A/B: PCG iterations as a replayed CUDA graph (default) vs plain launches (HWG_GRAPH=0)
for c in 2 4; do
  for v in 1 0 1 0; do
    HWG_GRAPH=$v python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg$c graph=$v', d['time_to_solve_s'], d['config']['iterations_per_solve'], d['gpu_launches'], d['e2e']['time_to_solve_s'])"
  done
done
