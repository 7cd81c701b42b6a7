python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r4j_build.log 2>&1
run() { tag=$1; L=$2; shift 2
  SS_LIB=$L timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-full-parity "$@" > gpurun_out/r4j_$tag.json 2> gpurun_out/r4j_$tag.err
  echo "$tag $(python -c "import json;d=json.load(open('gpurun_out/r4j_$tag.json'));print(d['ms_per_phase']['transfer_apply'], d['ms_per_step'], d['bit_exact_replica'])")" >> gpurun_out/r4j_all.txt
}
B=paper_2605_07330_b200/build
for i in 1 2; do
  for v in cur2 fd43 fd42 fd34; do run r10_${v}_$i $B/libsparsesync_$v.so --rho 0.1 --replica snapshot --steps 5; done
  for v in cur2 fd43 fd42 fd34; do run r05_${v}_$i $B/libsparsesync_$v.so --rho 0.05 --replica snapshot --steps 5; done
done
