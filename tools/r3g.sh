python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r3g_build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r3g_pytest.log 2>&1
run() { tag=$1; L=$2; shift 2
  SS_LIB=$L timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-full-parity "$@" > gpurun_out/r3g_$tag.json 2> gpurun_out/r3g_$tag.err
  echo "$tag $(python -c "import json;d=json.load(open('gpurun_out/r3g_$tag.json'));print(d['ms_per_phase']['compress_pack'], d['ms_per_step'])")" >> gpurun_out/r3g_all.txt
}
B=paper_2605_07330_b200/build
for i in 1 2 3; do
  run r01_head$i $B/libsparsesync_head.so --steps 10
  run r01_new$i "" --steps 10
done
for i in 1 2; do
  run r10_head$i $B/libsparsesync_head.so --rho 0.1 --replica snapshot --steps 5
  run r10_new$i "" --rho 0.1 --replica snapshot --steps 5
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_encode" -s 1 -c 1 -o gpurun_out/r3g_enc python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-full-parity --no-verify --latency-steps 0 > gpurun_out/r3g_ncu.log 2>&1
