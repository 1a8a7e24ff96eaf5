#!/bin/bash
# C5 16 GiB at 2 MiB pages: K1 5.49 in r2zu vs 5.90 in r2zf -- merge / hooks A/B
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2zv_build.log 2>&1
for k in 1 2; do for M in 1 0; do for H in 0 1; do
GCR_SCAN_MERGE=$M GCR_K1_HOOKS=$H timeout 600 python bench.py --no-cpu-baseline --sub-c4-gib 0 --config C5 --gib 16 --page-size 2097152 --compress 0 --steps 3 > gpurun_out/r2zv_m${M}_h${H}_$k.json 2>/dev/null
done; done; done
