python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2l_build.log 2>&1
for v in base e8u4 e7u6 s2k base; do
  if [ $v = base ]; then L=""; else L="paper_2605_07330_b200/build/libsparsesync_$v.so"; fi
  SS_LIB=$L timeout 600 python bench.py --no-full-parity --no-e2e --no-cpu-baseline > gpurun_out/r2l_${v}_r01.json 2> gpurun_out/r2l_${v}_r01.err
  SS_LIB=$L timeout 600 python bench.py --no-full-parity --no-e2e --no-cpu-baseline --rho 0.1 --replica snapshot > gpurun_out/r2l_${v}_r10.json 2> gpurun_out/r2l_${v}_r10.err
done
