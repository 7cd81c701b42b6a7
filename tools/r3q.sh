python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r3q_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_tracking.py tests/test_gpu_parity.py tests/test_gpu_scale.py tests/test_gpu_guard.py -x -q > gpurun_out/r3q_pytest.log 2>&1
run() { tag=$1; L=$2; shift 2
  SS_LIB=$L timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-full-parity "$@" > gpurun_out/r3q_$tag.json 2> gpurun_out/r3q_$tag.err
  echo "$tag $(python -c "import json;d=json.load(open('gpurun_out/r3q_$tag.json'));print(d['ms_per_phase']['extract'], d['ms_per_step'], (d.get('latency_per_update') or {}).get('median_ms'))")" >> gpurun_out/r3q_all.txt
}
B=paper_2605_07330_b200/build
for i in 1 2; do
  run cast4b_base_$i $B/libsparsesync_base.so --workload qwen3-4b --tracking cast
  run cast4b_new_$i "" --workload qwen3-4b --tracking cast
done
P=30300
for v in base new; do
  if [ $v = new ]; then L=""; else L="$B/libsparsesync_base.so"; fi
  P=$((P+1)); SS_LIB=$L timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $P bench.py --gpus 2 --workload qwen3-235b-a22b --topology sharded --model-shards 4 --stream-gb 5 --tracking cast --steps 5 --no-e2e > gpurun_out/r3q_cfg5_$v.json 2> gpurun_out/r3q_cfg5_$v.err
  echo "cfg5_$v $(python -c "import json;d=json.load(open('gpurun_out/r3q_cfg5_$v.json'));print(d['ms_per_phase'], d['ms_per_step'], (d.get('latency_per_update') or {}).get('median_ms'))")" >> gpurun_out/r3q_all.txt
done
