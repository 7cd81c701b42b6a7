python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r3m_build.log 2>&1
B="timeout 600 python bench.py --no-full-parity --no-e2e --no-cpu-baseline"
$B --rho 0.1 --replica snapshot > gpurun_out/r3m_r10.json 2> gpurun_out/r3m_r10.err
$B --commit scatter > gpurun_out/r3m_scatter.json 2> gpurun_out/r3m_scatter.err
$B --rho 0.001 > gpurun_out/r3m_r001.json 2> gpurun_out/r3m_r001.err
$B --dtype fp8 > gpurun_out/r3m_fp8.json 2> gpurun_out/r3m_fp8.err
$B --mask E --escape > gpurun_out/r3m_E_esc.json 2> gpurun_out/r3m_E_esc.err
$B --workload qwen3-4b --tracking cast > gpurun_out/r3m_cast4b.json 2> gpurun_out/r3m_cast4b.err
