python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2j_smoke.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2j_pytest.log 2>&1
timeout 600 python bench.py --no-full-parity > gpurun_out/r2j_bench.json 2> gpurun_out/r2j_bench.err
timeout 600 python bench.py --no-full-parity --no-e2e --no-cpu-baseline --rho 0.1 --replica snapshot > gpurun_out/r2j_bench_r10.json 2> gpurun_out/r2j_bench_r10.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_chunk_stats|k_encode|k_plan|k_bucket|k_pack|k_extract" -c 40 --csv --log-file gpurun_out/r2j_launches.csv python bench.py --steps 2 --warmup 3 --no-full-parity --no-e2e --no-cpu-baseline --no-verify --latency-steps 0 > gpurun_out/r2j_ncu.log 2>&1
SS_XPROF=1 timeout 600 python bench.py --workload 30b-slice --rho 0.1 --steps 2 --warmup 1 --no-full-parity --no-e2e --no-cpu-baseline --no-verify --latency-steps 0 > gpurun_out/r2j_xprof.json 2> gpurun_out/r2j_xprof.err
