python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2h_smoke.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2h_pytest.log 2>&1
timeout 600 python bench.py --no-full-parity > gpurun_out/r2h_bench.json 2> gpurun_out/r2h_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_chunk_stats|k_encode|k_plan|k_bucket|k_pack" -c 40 --csv --log-file gpurun_out/r2h_launches.csv python bench.py --steps 2 --warmup 3 --no-full-parity --no-e2e --no-cpu-baseline --no-verify --latency-steps 0 > gpurun_out/r2h_ncu.log 2>&1
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_run.py > gpurun_out/r2h_memcheck.log 2>&1
timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python tools/sanitize_run.py --small > gpurun_out/r2h_synccheck.log 2>&1
timeout 1200 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 20 python tools/sanitize_run.py --small > gpurun_out/r2h_racecheck.log 2>&1
