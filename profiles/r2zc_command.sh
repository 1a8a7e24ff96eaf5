#!/bin/bash
# K1g immediate-base braid (no per-lookup IADD; probe-verified smem base):
# K1g parity + verify tests, same-box A/B (GCR_GRP_IMM=0/1) on C2 at 4 KiB and
# 8 KiB pages and C5 16 GiB at 4 KiB; ncu of the new K1g
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2zc_smoke.log 2>&1
GCR_TRACE=1 python -c "
import torch; from paper_2502_16631_b200 import gcr; c=gcr.Context(0); c.close()" > gpurun_out/r2zc_probe.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_verify.py tests/test_gpu_codec.py -m gpu -q -x -k "4096 or 8192 or small or grp" > gpurun_out/r2zc_tests.log 2>&1; echo rc=$? >> gpurun_out/r2zc_tests.log
for k in 1 2; do for I in 1 0; do
GCR_GRP_IMM=$I timeout 600 python bench.py --no-cpu-baseline --sub-c4-gib 0 --page-size 4096 --compress 0 --steps 5 > gpurun_out/r2zc_c2p4k_imm${I}_$k.json 2>/dev/null
GCR_GRP_IMM=$I timeout 600 python bench.py --no-cpu-baseline --sub-c4-gib 0 --page-size 8192 --compress 0 --steps 5 > gpurun_out/r2zc_c2p8k_imm${I}_$k.json 2>/dev/null
GCR_GRP_IMM=$I timeout 600 python bench.py --no-cpu-baseline --sub-c4-gib 0 --config C5 --gib 16 --page-size 4096 --compress 0 --steps 3 > gpurun_out/r2zc_c5p4k_imm${I}_$k.json 2>/dev/null
done; done
NCU="ncu --set full --clock-control none --import-source on"
timeout 900 $NCU -k regex:k_scan_grp -c 2 -o gpurun_out/r2zc_grp python bench.py --steps 1 --warmup 0 --no-cpu-baseline --sub-c4-gib 0 --compress 0 --page-size 4096 > gpurun_out/r2zc_ncu.log 2>&1
