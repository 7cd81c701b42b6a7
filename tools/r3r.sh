python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r3r_build.log 2>&1
P=30400
for sg in 5 10 20 40; do
  P=$((P+1)); timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $P bench.py --gpus 2 --workload qwen3-235b-a22b --topology sharded --model-shards 4 --stream-gb $sg --tracking cast --steps 5 --no-e2e > gpurun_out/r3r_cfg5_sg$sg.json 2> gpurun_out/r3r_cfg5_sg$sg.err
  echo "sg$sg $(python -c "import json;d=json.load(open('gpurun_out/r3r_cfg5_sg$sg.json'));print(d['ms_per_phase'], d['ms_per_step'], d['latency_per_update']['median_ms'], d['config']['groups'])")" >> gpurun_out/r3r_all.txt
done
