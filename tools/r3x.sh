python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r3x_smoke.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -rs > gpurun_out/r3x_pytest.log 2>&1
timeout 900 python bench.py > gpurun_out/r3x_bench.json 2> gpurun_out/r3x_bench.err
