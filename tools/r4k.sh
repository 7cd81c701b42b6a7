python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r4k_smoke.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -rs > gpurun_out/r4k_pytest.log 2>&1
B="timeout 600 python bench.py --no-full-parity --no-e2e --no-cpu-baseline"
for t in "r10 --rho 0.1 --replica snapshot" "r05 --rho 0.05 --replica snapshot" "f8r10 --rho 0.1 --dtype fp8" "r01" "4b24 --workload qwen3-4b --groups 24"; do set -- $t; tag=$1; shift
  $B "$@" > gpurun_out/r4k_$tag.json 2> gpurun_out/r4k_$tag.err
  echo "$tag $(python -c "import json;d=json.load(open('gpurun_out/r4k_$tag.json'));print(d['ms_per_phase']['transfer_apply'], d['ms_per_step'], d['bit_exact_replica'])")" >> gpurun_out/r4k_all.txt
done
