python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r3e_build.log 2>&1
run() { # tag lib castw args...
  tag=$1; L=$2; C=$3; shift 3
  SS_LIB=$L SS_CASTW=$C timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-full-parity "$@" > gpurun_out/r3e_$tag.json 2> gpurun_out/r3e_$tag.err
  echo "$tag $(python -c "import json;d=json.load(open('gpurun_out/r3e_$tag.json'));print(d['ms_per_phase'], d['ms_per_step'])")" >> gpurun_out/r3e_all.txt
}
B=paper_2605_07330_b200/build
for i in 1 2; do
  run cast_head$i $B/libsparsesync_head.so 0 --workload qwen3-4b --tracking cast
  run cast_w0_$i "" 0 --workload qwen3-4b --tracking cast
  run cast_w1_$i "" 1 --workload qwen3-4b --tracking cast
  run cast_w2_$i "" 2 --workload qwen3-4b --tracking cast
done
for i in 1 2; do
  run cs_head$i $B/libsparsesync_head.so 0 --steps 10
  run cs_new$i "" 0 --steps 10
  run cs_w12_$i $B/libsparsesync_wpf12.so 0 --steps 10
  run cs_w16_$i $B/libsparsesync_wpf16.so 0 --steps 10
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_extract" -s 1 -c 1 -o gpurun_out/r3e_k1_r10 python bench.py --workload 30b-slice --rho 0.1 --replica snapshot --steps 1 --warmup 2 --no-e2e --no-cpu-baseline --no-full-parity --no-verify --latency-steps 0 > gpurun_out/r3e_ncu_k1.log 2>&1
