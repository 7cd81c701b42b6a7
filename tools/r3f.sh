python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r3f_build.log 2>&1
run() { tag=$1; L=$2; shift 2
  SS_LIB=$L timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-full-parity "$@" > gpurun_out/r3f_$tag.json 2> gpurun_out/r3f_$tag.err
  echo "$tag $(python -c "import json;d=json.load(open('gpurun_out/r3f_$tag.json'));print(d['ms_per_phase']['extract'], d['roofline']['frac'], d['ms_per_step'])")" >> gpurun_out/r3f_all.txt
}
B=paper_2605_07330_b200/build
for i in 1 2; do
  run r10_head$i $B/libsparsesync_head.so --rho 0.1 --replica snapshot --steps 5
  run r10_new$i "" --rho 0.1 --replica snapshot --steps 5
  run r10_x2_$i $B/libsparsesync_x2.so --rho 0.1 --replica snapshot --steps 5
done
for i in 1 2; do
  run r01_head$i $B/libsparsesync_head.so --steps 10
  run r01_new$i "" --steps 10
  run r01_x2_$i $B/libsparsesync_x2.so --steps 10
done
run f8r10_head $B/libsparsesync_head.so --rho 0.1 --replica snapshot --steps 5 --dtype fp8
run f8r10_new "" --rho 0.1 --replica snapshot --steps 5 --dtype fp8
run f8r10_x2 $B/libsparsesync_x2.so --rho 0.1 --replica snapshot --steps 5 --dtype fp8
