python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r4e_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py tests/test_gpu_guard.py -x -q > gpurun_out/r4e_pytest.log 2>&1
run() { tag=$1; L=$2; shift 2
  SS_LIB=$L timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-full-parity "$@" > gpurun_out/r4e_$tag.json 2> gpurun_out/r4e_$tag.err
  echo "$tag $(python -c "import json;d=json.load(open('gpurun_out/r4e_$tag.json'));print(d['ms_per_phase']['transfer_apply'], d['ms_per_step'], d['bit_exact_replica'])")" >> gpurun_out/r4e_all.txt
}
B=paper_2605_07330_b200/build
for i in 1 2; do
  for v in nofast fast; do L=""; [ $v = nofast ] && L=$B/libsparsesync_nofast.so
    run 4b24_${v}_$i "$L" --workload qwen3-4b --groups 24 --steps 10
    run 4b_${v}_$i "$L" --workload qwen3-4b --steps 10
    run r01_${v}_$i "$L" --steps 10
    run r10_${v}_$i "$L" --rho 0.1 --replica snapshot --steps 5
  done
done
P=31000
for v in nofast fast; do L=""; [ $v = nofast ] && L=$B/libsparsesync_nofast.so; P=$((P+1))
  SS_LIB=$L timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $P bench.py --gpus 2 --workload qwen3-4b --topology pair --no-e2e > gpurun_out/r4e_pair4b_$v.json 2> gpurun_out/r4e_pair4b_$v.err
  echo "pair4b_$v $(python -c "import json;d=json.load(open('gpurun_out/r4e_pair4b_$v.json'));print(d['ms_per_step'], d['latency_per_update']['median_ms'])")" >> gpurun_out/r4e_all.txt
  P=$((P+1))
  SS_LIB=$L timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $P bench.py --gpus 2 --workload qwen3-235b-a22b --topology sharded --model-shards 4 --stream-gb 10 --tracking cast --steps 5 --no-e2e > gpurun_out/r4e_cfg5_$v.json 2> gpurun_out/r4e_cfg5_$v.err
  echo "cfg5_$v $(python -c "import json;d=json.load(open('gpurun_out/r4e_cfg5_$v.json'));print(d['ms_per_step'], d['latency_per_update']['median_ms'])")" >> gpurun_out/r4e_all.txt
done
