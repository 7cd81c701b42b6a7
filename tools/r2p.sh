python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2p_build.log 2>&1
for w in 3 4 3 4; do for r in 0.01 0.1; do
  SS_XWRITERS=$w timeout 600 python bench.py --no-full-parity --no-e2e --no-cpu-baseline --rho $r --replica snapshot --no-verify > gpurun_out/r2p_w${w}_r$r.json 2> gpurun_out/r2p_w${w}_r$r.err
  echo "w=$w rho=$r $(cat gpurun_out/r2p_w${w}_r$r.json)" >> gpurun_out/r2p_all.txt
done; done
timeout 300 tools/scatter_bench 8589934592 0.01 > gpurun_out/r2p_scatter.txt 2>&1
timeout 300 tools/scatter_bench 8589934592 0.1 >> gpurun_out/r2p_scatter.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:"k_scatter_sector|k_scatter_strided" -c 12 --csv --log-file gpurun_out/r2p_scatter_ncu.csv tools/scatter_bench 8589934592 0.01 > /dev/null 2>&1
