python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2ff_build.log 2>&1
B="timeout 600 python bench.py --no-full-parity --no-e2e --no-cpu-baseline"
$B > gpurun_out/r2ff_base.json 2> gpurun_out/r2ff_base.err
$B --groups 2 --decode-pipeline > gpurun_out/r2ff_dp2.json 2> gpurun_out/r2ff_dp2.err
$B --groups 4 --decode-pipeline > gpurun_out/r2ff_dp4.json 2> gpurun_out/r2ff_dp4.err
$B --groups 8 --decode-pipeline > gpurun_out/r2ff_dp8.json 2> gpurun_out/r2ff_dp8.err
$B > gpurun_out/r2ff_base2.json 2> gpurun_out/r2ff_base2.err
