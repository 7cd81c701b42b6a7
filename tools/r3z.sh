python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r3z_build.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" -c 2000 --csv --log-file gpurun_out/r3z_4b_g24.csv python bench.py --workload qwen3-4b --groups 24 --steps 1 --warmup 3 --no-full-parity --no-e2e --no-cpu-baseline --no-verify --latency-steps 0 > gpurun_out/r3z_ncu.log 2>&1
P=30900
for g in 1 2 4; do P=$((P+1));
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $P bench.py --gpus 2 --workload qwen3-4b --topology pair --groups $g --no-e2e > gpurun_out/r3z_pair4b_g$g.json 2> gpurun_out/r3z_pair4b_g$g.err
  echo "pair4b g$g $(python -c "import json;d=json.load(open('gpurun_out/r3z_pair4b_g$g.json'));print(d['ms_per_step'], d['latency_per_update']['median_ms'])")" >> gpurun_out/r3z_all.txt
done
