python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2q_smoke.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2q_pytest.log 2>&1
timeout 900 python bench.py > gpurun_out/r2q_bench.json 2> gpurun_out/r2q_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/r2q_ref.json 2> gpurun_out/r2q_ref.err
timeout 600 python bench.py --no-full-parity --no-e2e --no-cpu-baseline --dtype fp8 > gpurun_out/r2q_fp8.json 2> gpurun_out/r2q_fp8.err
timeout 600 python bench.py --no-full-parity --no-e2e --no-cpu-baseline --rho 0.1 --replica snapshot > gpurun_out/r2q_r10.json 2> gpurun_out/r2q_r10.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2q_launches.csv python bench.py --steps 2 --warmup 3 --no-full-parity --no-e2e --no-cpu-baseline --no-verify --latency-steps 0 > gpurun_out/r2q_ncu.log 2>&1
