python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r4l_smoke.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -rs > gpurun_out/r4l_pytest.log 2>&1
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py > gpurun_out/r4l_bench.json 2> gpurun_out/r4l_bench.err
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --impl reference > gpurun_out/r4l_ref.json 2> gpurun_out/r4l_ref.err
P=31300
run() { name=$1; n=$2; shift 2; P=$((P+1));
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $P bench.py --gpus $n "$@" > gpurun_out/r4l_$name.json 2> gpurun_out/r4l_$name.err; }
run ring2 2
run pair2_4b 2 --workload qwen3-4b --topology pair --no-e2e
run cfg5_f1 2 --workload qwen3-235b-a22b --topology sharded --model-shards 4 --stream-gb 10 --tracking cast --steps 5 --no-e2e
CUDA_VISIBLE_DEVICES=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_extract|k_chunk|k_plan|k_bucket|k_encode|k_pack|k_decode|k_commit|k_crc" -c 200 --csv --log-file gpurun_out/r4l_launches.csv python bench.py --steps 2 --warmup 3 --no-full-parity --no-e2e --no-cpu-baseline --no-verify --latency-steps 0 > gpurun_out/r4l_ncu.log 2>&1
