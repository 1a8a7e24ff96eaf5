#!/bin/bash
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 1000 --csv --log-file gpurun_out/r1f_launches_bench.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r1f_launch_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_scan -c 3 -o gpurun_out/r1f_kscan python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/r1f_ncu_kscan.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_pack|k_scatter|k_tile_scan|k_zero" -c 6 -o gpurun_out/r1f_kother python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/r1f_ncu_kother.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_scan -c 1 -o gpurun_out/r1f_kscan_c4 python bench.py --config C4 --gib 8 --mode incremental --dirty 0.01 --steps 1 --warmup 0 --chunk-mb 1024 --no-cpu-baseline > gpurun_out/r1f_ncu_kscan_c4.log 2>&1
ls -la gpurun_out
