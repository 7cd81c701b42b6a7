python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2bb_build.log 2>&1
P=29900
run() { name=$1; n=$2; shift 2; P=$((P+1));
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $P bench.py --gpus $n "$@" > gpurun_out/r2bb_$name.json 2> gpurun_out/r2bb_$name.err; }
run fanout4_a 4 --topology fanout --no-e2e
run fanout4_b 4 --topology fanout --no-e2e --steps 20
run sharded4_a 4 --topology sharded --no-e2e --steps 20
run ring4 4
