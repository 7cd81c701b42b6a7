python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r3c_build.log 2>&1
for v in head new; do
  if [ $v = new ]; then L=""; else L="paper_2605_07330_b200/build/libsparsesync_$v.so"; fi
  SS_LIB=$L timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_chunk_stats|k_encode" -s 2 -c 2 -o gpurun_out/r3c_cs_$v python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-full-parity --no-verify --latency-steps 0 > gpurun_out/r3c_ncu_$v.log 2>&1
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_cast_track" -s 1 -c 1 -o gpurun_out/r3c_cast python bench.py --workload qwen3-4b --tracking cast --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-full-parity --no-verify --latency-steps 0 > gpurun_out/r3c_ncu_cast.log 2>&1
