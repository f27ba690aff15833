# round-end evidence: GPU tests, smoke, default bench (cfg 4), the reference arm,
# and a full ncu capture of the dominant kernel (finest-level UP pass, K = 10)
python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo rc=$? >> gpurun_out/smoke.log
python bench.py > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err
python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
bash scripts/ncu_up.sh
ncu -i gpurun_out/ncu_up.ncu-rep --page details > gpurun_out/ncu_up_details.txt 2>/dev/null
