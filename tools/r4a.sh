python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r4a_build.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_decode|k_chunk_stats" -s 60 -c 2 -o gpurun_out/r4a_small python bench.py --workload qwen3-4b --groups 24 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-full-parity --no-verify --latency-steps 0 > gpurun_out/r4a_ncu.log 2>&1
