set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2g_smoke.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2g_pytest.log 2>&1
timeout 600 python bench.py --no-full-parity > gpurun_out/r2g_bench.json 2> gpurun_out/r2g_bench.err
timeout 600 python bench.py --no-full-parity --no-e2e --no-cpu-baseline --rho 0.1 --replica snapshot > gpurun_out/r2g_bench_r10.json 2> gpurun_out/r2g_bench_r10.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_chunk_stats|k_encode|k_plan|k_bucket|k_pack" -c 40 --csv --log-file gpurun_out/r2g_launches.csv python bench.py --steps 2 --warmup 3 --no-full-parity --no-e2e --no-cpu-baseline --no-verify --latency-steps 0 > gpurun_out/r2g_ncu.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed --clock-control none --csv --log-file gpurun_out/r2g_scatter_ncu.csv tools/scatter_bench 8589934592 0.01 > gpurun_out/r2g_scatter.log 2>&1
