#!/bin/bash
# source-level ncu of K1g (4 KiB pages) and K1 (64 KiB) on C2: per-line
# instruction / stall attribution of the per-group overhead
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2zb_build.log 2>&1
NCU="ncu --set full --clock-control none --import-source on"
timeout 900 $NCU -k regex:k_scan_grp -c 2 -o gpurun_out/r2zb_grp python bench.py --steps 1 --warmup 0 --no-cpu-baseline --sub-c4-gib 0 --compress 0 --page-size 4096 > gpurun_out/r2zb_ncu1.log 2>&1
timeout 900 $NCU -k regex:k_scan -c 2 -o gpurun_out/r2zb_k1 python bench.py --steps 1 --warmup 0 --no-cpu-baseline --sub-c4-gib 0 --compress 0 > gpurun_out/r2zb_ncu2.log 2>&1
