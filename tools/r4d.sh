python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r4d_build.log 2>&1
run() { tag=$1; shift
  timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-full-parity "$@" > gpurun_out/r4d_$tag.json 2> gpurun_out/r4d_$tag.err
  echo "$tag $(python -c "import json;d=json.load(open('gpurun_out/r4d_$tag.json'));print(d['ms_per_step'], d['ms_per_phase'], d['bit_exact_replica'])")" >> gpurun_out/r4d_all.txt
}
for i in 1 2; do
  run base_$i
  SS_DCTAS=256 run dp2_c256_$i --decode-pipeline --groups 2
  SS_DCTAS=236 run dp4_c236_$i --decode-pipeline --groups 4
  SS_DCTAS=256 run dp4_c256_$i --decode-pipeline --groups 4
  SS_DCTAS=200 run dp4_c200_$i --decode-pipeline --groups 4
  run dp4_nocap_$i --decode-pipeline --groups 4
  SS_DCTAS=256 run base_c256_$i
done
