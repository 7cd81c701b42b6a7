python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r3p_smoke.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q -rs > gpurun_out/r3p_pytest.log 2>&1
B="timeout 600 python bench.py --no-full-parity --no-e2e --no-cpu-baseline"
$B --rho 0.1 --replica snapshot > gpurun_out/r3p_r10.json 2> gpurun_out/r3p_r10.err
$B --rho 0.1 --dtype fp8 > gpurun_out/r3p_f8r10.json 2> gpurun_out/r3p_f8r10.err
$B --rho 0.05 --replica snapshot > gpurun_out/r3p_r05.json 2> gpurun_out/r3p_r05.err
$B > gpurun_out/r3p_r01.json 2> gpurun_out/r3p_r01.err
