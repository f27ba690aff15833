# A/B: coarse-level MG arithmetic below the streamed levels (exact vs fast)
for v in 1 0 1 0; do
  HWG_COARSE_EXACT=$v python bench.py --config 2 --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('exact=$v', d['time_to_solve_s'], d['config']['iterations_per_solve'], d['kernel_classes_ms']['mg2d_coarse'])"
done
