python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2ee_build.log 2>&1
for r in 0.1 0.01; do
SS_XPROF=1 timeout 600 python bench.py --workload 30b-slice --rho $r --steps 2 --warmup 1 --no-full-parity --no-e2e --no-cpu-baseline --no-verify --latency-steps 0 > /dev/null 2> gpurun_out/r2ee_xprof_$r.err
done
SS_XPROF=1 SS_XWRITERS=3 timeout 600 python bench.py --workload 30b-slice --rho 0.1 --steps 2 --warmup 1 --no-full-parity --no-e2e --no-cpu-baseline --no-verify --latency-steps 0 > /dev/null 2> gpurun_out/r2ee_xprof_w3.err
