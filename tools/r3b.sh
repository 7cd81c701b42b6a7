python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r3b_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -x -q > gpurun_out/r3b_pytest.log 2>&1
for v in head new head new; do
  if [ $v = new ]; then L=""; else L="paper_2605_07330_b200/build/libsparsesync_$v.so"; fi
  SS_LIB=$L timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-full-parity --steps 10 > gpurun_out/r3b_$v.json 2> gpurun_out/r3b_$v.err
  echo "$v $(python -c "import json;d=json.load(open('gpurun_out/r3b_$v.json'));print(d['ms_per_phase'], d['ms_per_step'])")" >> gpurun_out/r3b_all.txt
done
for v in head new; do
  if [ $v = new ]; then L=""; else L="paper_2605_07330_b200/build/libsparsesync_$v.so"; fi
  SS_LIB=$L timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-full-parity --rho 0.1 --replica snapshot --steps 5 > gpurun_out/r3b_r10_$v.json 2> gpurun_out/r3b_r10_$v.err
  echo "r10 $v $(python -c "import json;d=json.load(open('gpurun_out/r3b_r10_$v.json'));print(d['ms_per_phase'], d['ms_per_step'])")" >> gpurun_out/r3b_all.txt
done
