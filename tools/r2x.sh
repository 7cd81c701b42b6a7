python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2x_build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_tracking.py -q > gpurun_out/r2x_pytest_tracking.log 2>&1
for v in old new old new; do
  if [ $v = new ]; then L=""; else L="paper_2605_07330_b200/build/libsparsesync_$v.so"; fi
  SS_LIB=$L timeout 600 python bench.py --workload qwen3-4b --tracking cast --no-e2e --no-cpu-baseline --no-full-parity > gpurun_out/r2x_cast_$v.json 2> gpurun_out/r2x_cast_$v.err
  echo "$v $(cat gpurun_out/r2x_cast_$v.json)" >> gpurun_out/r2x_all.txt
done
