python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r3d_build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_tracking.py -x -q > gpurun_out/r3d_pytest_track.log 2>&1
SS_CAST=direct timeout 600 python -m pytest tests/test_gpu_tracking.py -x -q > gpurun_out/r3d_pytest_track_direct.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/r3d_pytest_parity.log 2>&1
run() { # tag lib cast args...
  tag=$1; L=$2; C=$3; shift 3
  SS_LIB=$L SS_CAST=$C timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-full-parity "$@" > gpurun_out/r3d_$tag.json 2> gpurun_out/r3d_$tag.err
  echo "$tag $(python -c "import json;d=json.load(open('gpurun_out/r3d_$tag.json'));print(d['ms_per_phase'], d['ms_per_step'])")" >> gpurun_out/r3d_all.txt
}
H=paper_2605_07330_b200/build/libsparsesync_head.so
for i in 1 2; do
  run cast_head$i $H tma --workload qwen3-4b --tracking cast
  run cast_tma$i "" tma --workload qwen3-4b --tracking cast
  run cast_direct$i "" direct --workload qwen3-4b --tracking cast
done
for i in 1 2; do
  run cs_head$i $H tma --steps 10
  run cs_new$i "" tma --steps 10
done
