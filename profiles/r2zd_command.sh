#!/bin/bash
# round-2 final evidence on the current code: smoke, every GPU test, the
# default bench line (with cpu_baseline), the reference arm, 2 ranks on the
# 1-GPU box, the ncu launch list of the default bench and full captures of
# k_scan (C2), k_scan_grp (C2 at 4 KiB, after the probe launches), the TMA
# scatter + zero fill, the codec
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2zd_smoke.log 2>&1
timeout 2700 python -m pytest tests -m gpu -q > gpurun_out/r2zd_gputests.log 2>&1; echo rc=$? >> gpurun_out/r2zd_gputests.log
timeout 900 python bench.py > gpurun_out/r2zd_bench.json 2> gpurun_out/r2zd_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/r2zd_bench_ref.json 2> gpurun_out/r2zd_bench_ref.err
timeout 600 python bench.py --gpus 2 --steps 5 --no-cpu-baseline --sub-c4-gib 0 > gpurun_out/r2zd_bench_2ranks.json 2> gpurun_out/r2zd_bench_2ranks.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r2zd_launches_bench.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --sub-c4-gib 0 > gpurun_out/r2zd_launch_bench.log 2>&1
NCU="ncu --set full --clock-control none --import-source on"
$NCU -k regex:k_scan -c 2 -o gpurun_out/r2zd_kscan python bench.py --steps 1 --warmup 0 --no-cpu-baseline --sub-c4-gib 0 > gpurun_out/r2zd_ncu1.log 2>&1
$NCU -k regex:k_scan_grp --launch-skip 2 -c 2 -o gpurun_out/r2zd_kgrp python bench.py --steps 1 --warmup 0 --no-cpu-baseline --sub-c4-gib 0 --compress 0 --page-size 4096 > gpurun_out/r2zd_ncu2.log 2>&1
$NCU -k regex:"k_scatter|k_zero_fill|k_pack" -c 8 -o gpurun_out/r2zd_k4k6k7 python bench.py --steps 1 --warmup 0 --no-cpu-baseline --sub-c4-gib 0 --compress 0 --direct-min-mb -1 > gpurun_out/r2zd_ncu3.log 2>&1
$NCU -k regex:"k_codec" -c 8 -o gpurun_out/r2zd_codec python bench.py --steps 1 --warmup 0 --no-cpu-baseline --sub-c4-gib 0 > gpurun_out/r2zd_ncu4.log 2>&1
