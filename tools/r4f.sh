python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r4f_smoke.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -rs > gpurun_out/r4f_pytest.log 2>&1
run() { tag=$1; L=$2; shift 2
  SS_LIB=$L timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-full-parity "$@" > gpurun_out/r4f_$tag.json 2> gpurun_out/r4f_$tag.err
  echo "$tag $(python -c "import json;d=json.load(open('gpurun_out/r4f_$tag.json'));print(d['ms_per_phase']['transfer_apply'], d['ms_per_step'], d['bit_exact_replica'])")" >> gpurun_out/r4f_all.txt
}
B=paper_2605_07330_b200/build
for i in 1 2; do
  for v in nofast fast; do L=""; [ $v = nofast ] && L=$B/libsparsesync_nofast.so
    run 4b24_${v}_$i "$L" --workload qwen3-4b --groups 24 --steps 10
    run r10_${v}_$i "$L" --rho 0.1 --replica snapshot --steps 5
    run r001_${v}_$i "$L" --rho 0.001 --steps 10
  done
done
timeout 900 python bench.py > gpurun_out/r4f_bench.json 2> gpurun_out/r4f_bench.err
