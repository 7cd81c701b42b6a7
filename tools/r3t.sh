python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r3t_build.log 2>&1
P=30600
run() { name=$1; n=$2; shift 2; P=$((P+1));
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $P bench.py --gpus $n "$@" > gpurun_out/r3t_$name.json 2> gpurun_out/r3t_$name.err
  echo "$name $(python -c "import json;d=json.load(open('gpurun_out/r3t_$name.json'));print(d['ms_per_phase']['extract'], d['ms_per_phase']['compress_pack'], d['ms_per_step'], d['latency_per_update']['median_ms'], d['config']['groups'])")" >> gpurun_out/r3t_all.txt; }
for i in 1 2; do
  for df in 0 1; do
    SS_BENCH_DEFER=$df run cfg5_sg5_d${df}_$i 2 --workload qwen3-235b-a22b --topology sharded --model-shards 4 --stream-gb 5 --tracking cast --steps 5 --no-e2e
    SS_BENCH_DEFER=$df run cfg5_sg10_d${df}_$i 2 --workload qwen3-235b-a22b --topology sharded --model-shards 4 --stream-gb 10 --tracking cast --steps 5 --no-e2e
    SS_BENCH_DEFER=$df run pair4b_d${df}_$i 2 --workload qwen3-4b --topology pair --no-e2e
    SS_BENCH_DEFER=$df run pair30b_d${df}_$i 2 --topology pair --no-e2e
  done
done
