python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2n_build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -x -q > gpurun_out/r2n_pytest.log 2>&1
for v in old new old new; do
  if [ $v = new ]; then L=""; else L="paper_2605_07330_b200/build/libsparsesync_$v.so"; fi
  SS_LIB=$L timeout 600 python bench.py --no-full-parity --no-e2e --no-cpu-baseline --steps 20 > gpurun_out/r2n_${v}_r01.json 2> gpurun_out/r2n_${v}_r01.err
  cat gpurun_out/r2n_${v}_r01.json >> gpurun_out/r2n_all.jsonl
done
SS_LIB= timeout 600 python bench.py --no-full-parity --no-e2e --no-cpu-baseline --rho 0.1 --replica snapshot > gpurun_out/r2n_new_r10.json 2> gpurun_out/r2n_new_r10.err
