python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r4g_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -x -q > gpurun_out/r4g_pytest.log 2>&1
run() { tag=$1; L=$2; shift 2
  SS_LIB=$L timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-full-parity "$@" > gpurun_out/r4g_$tag.json 2> gpurun_out/r4g_$tag.err
  echo "$tag $(python -c "import json;d=json.load(open('gpurun_out/r4g_$tag.json'));print(d['ms_per_phase']['transfer_apply'], d['ms_per_step'], d['bit_exact_replica'])")" >> gpurun_out/r4g_all.txt
}
B=paper_2605_07330_b200/build
for i in 1 2; do
  for v in head3 new; do L=""; [ $v = head3 ] && L=$B/libsparsesync_head3.so
    run 4b24_${v}_$i "$L" --workload qwen3-4b --groups 24 --steps 10
    run r01_${v}_$i "$L" --steps 10
    run r10_${v}_$i "$L" --rho 0.1 --replica snapshot --steps 5
  done
done
