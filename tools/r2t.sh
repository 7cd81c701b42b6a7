python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2t_build.log 2>&1
B="timeout 600 python bench.py --no-full-parity --no-e2e --no-cpu-baseline"
$B > gpurun_out/r2t_base.json 2> gpurun_out/r2t_base.err
$B --groups 4 > gpurun_out/r2t_g4.json 2> gpurun_out/r2t_g4.err
$B --groups 4 --overlap-apply > gpurun_out/r2t_g4_ov.json 2> gpurun_out/r2t_g4_ov.err
$B --groups 8 --overlap-apply > gpurun_out/r2t_g8_ov.json 2> gpurun_out/r2t_g8_ov.err
SS_XCTAS=256 $B --groups 4 --overlap-apply > gpurun_out/r2t_g4_ov_x256.json 2> gpurun_out/r2t_g4_ov_x256.err
SS_XCTAS=220 $B --groups 4 --overlap-apply > gpurun_out/r2t_g4_ov_x220.json 2> gpurun_out/r2t_g4_ov_x220.err
SS_XCTAS=180 $B --groups 8 --overlap-apply > gpurun_out/r2t_g8_ov_x180.json 2> gpurun_out/r2t_g8_ov_x180.err
