#!/bin/bash
# round 2: CTA-shared f1 write-out; TMA K6/K7; 64 MiB restore groups.  Parity
# tests touched by these, then same-box A/B (f1 vs staged on C4 1 %, 5 %), C2
# bench default (compress) and uncompressed staged restore (K6)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2k_smoke.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_inscan.py tests/test_gpu_parity.py tests/test_gpu_codec.py tests/test_gpu_verify.py tests/test_gpu_stress.py -q -m gpu -x > gpurun_out/r2k_tests.log 2>&1; echo rc=$? >> gpurun_out/r2k_tests.log
OUT=gpurun_out/r2k_f1_ab.jsonl; : > $OUT
for rep in 1 2; do
for isp in 0 1; do
  for d in 0.01 0.05; do
    line=$(timeout 400 python bench.py --no-cpu-baseline --config C4 --mode incremental --dirty $d --steps 5 --compress 0 --in-scan-pack $isp 2> gpurun_out/r2k_c4_${isp}_${d}.err | tail -1)
    echo "{\"rep\": $rep, \"in_scan_pack\": $isp, \"dirty\": $d, \"line\": $line}" >> $OUT
  done
done
done
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r2k_bench.json 2> gpurun_out/r2k_bench.err
timeout 600 python bench.py --no-cpu-baseline --compress 0 --direct-min-mb -1 --steps 5 > gpurun_out/r2k_bench_staged.json 2> gpurun_out/r2k_bench_staged.err
