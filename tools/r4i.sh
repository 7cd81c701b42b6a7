python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r4i_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_nccl.py tests/test_gpu_peer.py -q -rs > gpurun_out/r4i_pytest_multi.log 2>&1
P=31200
run() { name=$1; n=$2; shift 2; P=$((P+1));
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $P bench.py --gpus $n "$@" > gpurun_out/r4i_$name.json 2> gpurun_out/r4i_$name.err; }
run ring4 4
run fanout4 4 --topology fanout --no-e2e
run sharded4 4 --topology sharded --no-e2e
run cfg5_f1_4 4 --workload qwen3-235b-a22b --topology sharded --model-shards 4 --stream-gb 10 --tracking cast --steps 5 --no-e2e
