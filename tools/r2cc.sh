python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2cc_smoke.log 2>&1
timeout 900 python -m pytest tests/test_gpu_scale.py -x -q > gpurun_out/r2cc_pytest_scale.log 2>&1
B="timeout 600 python bench.py --no-full-parity --no-e2e --no-cpu-baseline"
$B --workload 1m --steps 100 --warmup 10 > gpurun_out/r2cc_1m.json 2> gpurun_out/r2cc_1m.err
$B --workload 1m --steps 100 --warmup 10 --graph > gpurun_out/r2cc_1m_graph.json 2> gpurun_out/r2cc_1m_graph.err
$B --workload qwen3-4b > gpurun_out/r2cc_4b.json 2> gpurun_out/r2cc_4b.err
$B --workload qwen3-4b --graph > gpurun_out/r2cc_4b_graph.json 2> gpurun_out/r2cc_4b_graph.err
$B > gpurun_out/r2cc_30b.json 2> gpurun_out/r2cc_30b.err
$B --graph > gpurun_out/r2cc_30b_graph.json 2> gpurun_out/r2cc_30b_graph.err
