# round-end evidence: GPU tests, smoke, default bench (cfg 4), the reference arm,
# cfg 2 / cfg 3 / cfg 5-share bench lines
python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo rc=$? >> gpurun_out/smoke.log
python bench.py > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err
python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
python bench.py --config 2 --steps 5 > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
python bench.py --config 3 --steps 2 > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err
python bench.py --config 5 --steps 2 > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err
