python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2m_build.log 2>&1
nvidia-smi topo -m > gpurun_out/r2m_topo.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_nccl.py tests/test_gpu_peer.py -x -q -rs > gpurun_out/r2m_pytest_2gpu.log 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 > gpurun_out/r2m_bench_n2.json 2> gpurun_out/r2m_bench_n2.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --topology pair --no-e2e > gpurun_out/r2m_bench_n2_pair.json 2> gpurun_out/r2m_bench_n2_pair.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --topology pair --transport nccl --no-e2e > gpurun_out/r2m_bench_n2_pair_nccl.json 2> gpurun_out/r2m_bench_n2_pair_nccl.err
