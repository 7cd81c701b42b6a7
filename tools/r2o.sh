# 4-GPU box: NCCL data-plane tests at world 2 and 4, ring / fanout / sharded bench lines, config 5 (2 of 4 pairs)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2o_build.log 2>&1
nvidia-smi topo -m > gpurun_out/r2o_topo.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_nccl.py -q -rs > gpurun_out/r2o_pytest_nccl.log 2>&1
P=29600
run() { name=$1; n=$2; shift 2; P=$((P+1));
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $P bench.py --gpus $n "$@" > gpurun_out/r2o_$name.json 2> gpurun_out/r2o_$name.err; }
run ring2 2 --no-e2e
run ring4 4 --no-e2e
run fanout4_peer 4 --topology fanout --no-e2e
run fanout4_nccl 4 --topology fanout --transport nccl --no-e2e
run fanout4_bcast 4 --topology fanout --transport nccl-bcast --no-e2e
run sharded4 4 --topology sharded --no-e2e
run cfg5_235b 4 --workload qwen3-235b-a22b --topology sharded --model-shards 4 --stream-gb 5 --commit scatter --steps 5 --no-e2e
