#!/bin/bash
# round 2: every GPU test with f1 as the default incremental path; same-box A/B
# of the staged pipeline vs the in-scan pack on C4 (40 GiB, 1 % / 5 %); scan
# launch stamps with and without the entry prefetch
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2j_smoke.log 2>&1
timeout 2700 python -m pytest tests -m gpu -q > gpurun_out/r2j_gputests.log 2>&1; echo rc=$? >> gpurun_out/r2j_gputests.log
OUT=gpurun_out/r2j_f1_ab.jsonl; : > $OUT
for rep in 1 2; do
for isp in 0 1; do
  for d in 0.01 0.05; do
    line=$(timeout 400 python bench.py --no-cpu-baseline --config C4 --mode incremental --dirty $d --steps 5 --compress 0 --in-scan-pack $isp 2> gpurun_out/r2j_c4_${isp}_${d}.err | tail -1)
    echo "{\"rep\": $rep, \"in_scan_pack\": $isp, \"dirty\": $d, \"line\": $line}" >> $OUT
  done
done
done
GCR_SCAN_TIMES=1 timeout 300 python tools/scan_times.py 128 1024 > gpurun_out/r2j_scan_times.log 2>&1
GCR_SCAN_PREFETCH=0 GCR_SCAN_TIMES=1 timeout 300 python tools/scan_times.py 128 1024 > gpurun_out/r2j_scan_times_nopf.log 2>&1
