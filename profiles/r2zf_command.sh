#!/bin/bash
# the round-2 config sweep on the final code (tools/sweep.sh) + ncu of k_scan
# (exact kernel name: the K1g probe launches no longer match)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2zf_build.log 2>&1
NCU="ncu --set full --clock-control none --import-source on"
$NCU -k k_scan -c 2 -o gpurun_out/r2zf_kscan python bench.py --steps 1 --warmup 0 --no-cpu-baseline --sub-c4-gib 0 > gpurun_out/r2zf_ncu1.log 2>&1
bash tools/sweep.sh > gpurun_out/r2zf_sweep_stdout.txt 2>&1
cp gpurun_out/sweep.jsonl gpurun_out/r2zf_sweep.jsonl
