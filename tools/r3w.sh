python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r3w_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py tests/test_gpu_guard.py tests/test_gpu_tracking.py -x -q > gpurun_out/r3w_pytest.log 2>&1
run() { tag=$1; L=$2; shift 2
  SS_LIB=$L timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-full-parity "$@" > gpurun_out/r3w_$tag.json 2> gpurun_out/r3w_$tag.err
  echo "$tag $(python -c "import json;d=json.load(open('gpurun_out/r3w_$tag.json'));print(d['ms_per_phase']['compress_pack'], d['ms_per_step'])")" >> gpurun_out/r3w_all.txt
}
B=paper_2605_07330_b200/build
for i in 1 2; do
  for v in h0 h2 h3; do run r01_${v}_$i $B/libsparsesync_$v.so --steps 10; done
  for v in h0 h2 h3; do run 4b_${v}_$i $B/libsparsesync_$v.so --workload qwen3-4b --groups 24 --steps 10; done
  for v in h0 h2 h3; do run r10_${v}_$i $B/libsparsesync_$v.so --rho 0.1 --replica snapshot --steps 5; done
done
