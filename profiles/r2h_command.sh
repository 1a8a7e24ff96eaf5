#!/bin/bash
# round 2: f1 in-scan pack -- every GPU test (f1 is the default path of incremental
# checkpoints), then same-box A/B of the staged pipeline vs the in-scan pack on
# C4 (40 GiB, 1 % / 5 % dirty, incremental) and C2
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2h_smoke.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r2h_gputests.log 2>&1; echo rc=$? >> gpurun_out/r2h_gputests.log
OUT=gpurun_out/r2h_f1_ab.jsonl; : > $OUT
for rep in 1 2; do
for isp in 0 1; do
  for d in 0.01 0.05; do
    line=$(timeout 600 python bench.py --no-cpu-baseline --config C4 --mode incremental --dirty $d --steps 5 --compress 0 --in-scan-pack $isp 2> gpurun_out/r2h_c4_${isp}_${d}.err | tail -1)
    echo "{\"rep\": $rep, \"in_scan_pack\": $isp, \"dirty\": $d, \"line\": $line}" >> $OUT
  done
done
done
timeout 600 python bench.py --no-cpu-baseline --compress 0 --in-scan-pack 2 --steps 5 > gpurun_out/r2h_c2_isp2.json 2> gpurun_out/r2h_c2_isp2.err
