python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2aa_smoke.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py tests/test_gpu_guard.py -x -q > gpurun_out/r2aa_pytest.log 2>&1
for v in v0 new v0 new; do
  if [ $v = new ]; then L=""; else L="paper_2605_07330_b200/build/libsparsesync_$v.so"; fi
  for args in "--rho 0.01" "--rho 0.1 --replica snapshot" "--dtype fp8 --rho 0.1" "--dtype fp8"; do
    tag=$(echo $args | tr -d ' -')
    SS_LIB=$L timeout 600 python bench.py --no-full-parity --no-e2e --no-cpu-baseline --no-verify $args > gpurun_out/r2aa_${v}_$tag.json 2>/dev/null
    echo "$v $tag $(cat gpurun_out/r2aa_${v}_$tag.json)" >> gpurun_out/r2aa_all.txt
  done
done
