#!/bin/bash
# round 2: K1g raw16 table replicated 8x -- parity at 4/8 KiB, same-box A/B of
# C2 at 4 KiB pages (GCR_GRP_T4REP=0/1 alternating), ncu full captures of
# k_scan (64 KiB, 2 MiB), k_scan_grp (4 KiB, rep on/off), K6/K7 (TMA) and the
# codec kernels, plus the launch list of the default bench
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2l_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "4096 or 8192" > gpurun_out/r2l_tests.log 2>&1; echo rc=$? >> gpurun_out/r2l_tests.log
OUT=gpurun_out/r2l_t4rep_ab.jsonl; : > $OUT
for rep in 1 2 3; do
  for t in 0 1; do
    line=$(GCR_GRP_T4REP=$t timeout 300 python bench.py --no-cpu-baseline --sub-c4-gib 0 --compress 0 --page-size 4096 --steps 5 2> gpurun_out/r2l_t4rep_$t.err | tail -1)
    echo "{\"rep\": $rep, \"t4rep\": $t, \"line\": $line}" >> $OUT
  done
done
NCU="ncu --set full --clock-control none --import-source on"
$NCU -k regex:k_scan -c 2 -o gpurun_out/r2l_kscan python bench.py --steps 1 --warmup 0 --no-cpu-baseline --sub-c4-gib 0 --compress 0 > gpurun_out/r2l_ncu1.log 2>&1
$NCU -k regex:k_scan -c 2 -o gpurun_out/r2l_kscan_2m python bench.py --steps 1 --warmup 0 --no-cpu-baseline --sub-c4-gib 0 --compress 0 --page-size 2097152 > gpurun_out/r2l_ncu2.log 2>&1
GCR_GRP_T4REP=1 $NCU -k regex:k_scan_grp -c 2 -o gpurun_out/r2l_kscangrp_rep python bench.py --steps 1 --warmup 0 --no-cpu-baseline --sub-c4-gib 0 --compress 0 --page-size 4096 > gpurun_out/r2l_ncu3.log 2>&1
GCR_GRP_T4REP=0 $NCU -k regex:k_scan_grp -c 2 -o gpurun_out/r2l_kscangrp_norep python bench.py --steps 1 --warmup 0 --no-cpu-baseline --sub-c4-gib 0 --compress 0 --page-size 4096 > gpurun_out/r2l_ncu4.log 2>&1
$NCU -k regex:"k_scatter|k_zero_fill" -c 6 -o gpurun_out/r2l_k6k7 python bench.py --steps 1 --warmup 0 --no-cpu-baseline --sub-c4-gib 0 --compress 0 --direct-min-mb -1 > gpurun_out/r2l_ncu5.log 2>&1
$NCU -k regex:k_codec -c 8 -o gpurun_out/r2l_codec python bench.py --steps 1 --warmup 0 --no-cpu-baseline --sub-c4-gib 0 > gpurun_out/r2l_ncu6.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/r2l_launches_bench.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --sub-c4-gib 0 > gpurun_out/r2l_launch_bench.log 2>&1
