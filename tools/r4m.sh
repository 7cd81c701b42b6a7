python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r4m_build.log 2>&1
P=31400
for i in 1 2; do
for b in 256 128 64; do P=$((P+1))
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $P bench.py --gpus 2 --bucket-mb $b --no-e2e --no-cpu-baseline > gpurun_out/r4m_ring2_b$b.json 2> gpurun_out/r4m_ring2_b$b.err
  echo "ring2 b$b $(python -c "import json;d=json.load(open('gpurun_out/r4m_ring2_b$b.json'));print(d['value'], d['ms_per_step'], d['ms_per_phase']['transfer_apply'])")" >> gpurun_out/r4m_all.txt
  timeout 600 python bench.py --bucket-mb $b --no-e2e --no-cpu-baseline --no-full-parity > gpurun_out/r4m_one_b$b.json 2> gpurun_out/r4m_one_b$b.err
  echo "one b$b $(python -c "import json;d=json.load(open('gpurun_out/r4m_one_b$b.json'));print(d['value'], d['ms_per_step'], d['ms_per_phase']['transfer_apply'])")" >> gpurun_out/r4m_all.txt
done
done
