python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r3v_smoke.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -rs > gpurun_out/r3v_pytest.log 2>&1
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py > gpurun_out/r3v_bench.json 2> gpurun_out/r3v_bench.err
P=30700
run() { name=$1; n=$2; shift 2; P=$((P+1));
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $P bench.py --gpus $n "$@" > gpurun_out/r3v_$name.json 2> gpurun_out/r3v_$name.err; }
run ring2 2
run pair2_4b 2 --workload qwen3-4b --topology pair --no-e2e
run cfg5_f1 2 --workload qwen3-235b-a22b --topology sharded --model-shards 4 --stream-gb 10 --tracking cast --steps 5 --no-e2e
CUDA_VISIBLE_DEVICES=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_extract|k_chunk|k_plan|k_bucket|k_encode|k_pack|k_decode|k_commit|k_crc" -c 200 --csv --log-file gpurun_out/r3v_launches.csv python bench.py --steps 2 --warmup 3 --no-full-parity --no-e2e --no-cpu-baseline --no-verify --latency-steps 0 > gpurun_out/r3v_ncu.log 2>&1
CUDA_VISIBLE_DEVICES=0 timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_decode" -s 1 -c 1 -o gpurun_out/r3v_decode_r10 python bench.py --rho 0.1 --replica snapshot --workload 30b-slice --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-full-parity --no-verify --latency-steps 0 > gpurun_out/r3v_ncu_dec.log 2>&1
