python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r3a_smoke.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r3a_pytest.log 2>&1
timeout 900 python bench.py > gpurun_out/r3a_bench.json 2> gpurun_out/r3a_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/r3a_ref.json 2> gpurun_out/r3a_ref.err
timeout 900 python bench.py --dtype fp8 --no-full-parity > gpurun_out/r3a_fp8_e2e.json 2> gpurun_out/r3a_fp8_e2e.err
timeout 600 python bench.py --workload qwen3-4b --tracking cast --no-e2e --no-cpu-baseline --no-full-parity > gpurun_out/r3a_cast.json 2> gpurun_out/r3a_cast.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" -c 400 --csv --log-file gpurun_out/r3a_launches.csv python bench.py --steps 2 --warmup 3 --no-full-parity --no-e2e --no-cpu-baseline --no-verify --latency-steps 0 > gpurun_out/r3a_ncu.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_chunk_stats|k_encode" -s 2 -c 2 -o gpurun_out/r3a_compress python bench.py --workload 30b-slice --steps 1 --warmup 2 --no-e2e --no-cpu-baseline --no-full-parity --no-verify --latency-steps 0 > gpurun_out/r3a_ncu_compress.log 2>&1
