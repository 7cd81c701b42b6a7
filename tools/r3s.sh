python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r3s_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_peer.py tests/test_gpu_nccl.py -q -rs > gpurun_out/r3s_pytest.log 2>&1
P=30500
run() { name=$1; n=$2; shift 2; P=$((P+1));
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $P bench.py --gpus $n "$@" > gpurun_out/r3s_$name.json 2> gpurun_out/r3s_$name.err
  echo "$name $(python -c "import json;d=json.load(open('gpurun_out/r3s_$name.json'));print(d['ms_per_phase'], d['ms_per_step'], d['latency_per_update']['median_ms'], d['config']['groups'], d['bit_exact_replica'])")" >> gpurun_out/r3s_all.txt; }
run cfg5_sg5 2 --workload qwen3-235b-a22b --topology sharded --model-shards 4 --stream-gb 5 --tracking cast --steps 5 --no-e2e
run cfg5_sg10 2 --workload qwen3-235b-a22b --topology sharded --model-shards 4 --stream-gb 10 --tracking cast --steps 5 --no-e2e
run pair2_4b 2 --workload qwen3-4b --topology pair --no-e2e

run f1stream_4b 2 --workload qwen3-4b --topology sharded --stream-gb 1 --tracking cast --no-e2e
