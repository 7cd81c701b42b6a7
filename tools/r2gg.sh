python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2gg_build.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" -c 200 --csv --log-file gpurun_out/r2gg_1m_launches.csv python bench.py --workload 1m --steps 3 --warmup 3 --no-full-parity --no-e2e --no-cpu-baseline --no-verify --latency-steps 0 > gpurun_out/r2gg_ncu.log 2>&1
timeout 900 python bench.py --dtype fp8 --no-full-parity > gpurun_out/r2gg_fp8_e2e.json 2> gpurun_out/r2gg_fp8_e2e.err
