#!/bin/bash
# K1g raw16 table replicated x8 (GCR_GRP_T4REP=1) re-measured on the immediate-base kernel
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2zo_build.log 2>&1
for k in 1 2; do for T in 1 0; do
GCR_GRP_T4REP=$T timeout 600 python bench.py --no-cpu-baseline --sub-c4-gib 0 --page-size 4096 --compress 0 --steps 5 > gpurun_out/r2zo_c2p4k_t4rep${T}_$k.json 2>/dev/null
GCR_GRP_T4REP=$T timeout 600 python bench.py --no-cpu-baseline --sub-c4-gib 0 --config C5 --gib 16 --page-size 4096 --compress 0 --steps 3 > gpurun_out/r2zo_c5p4k_t4rep${T}_$k.json 2>/dev/null
done; done
GCR_GRP_T4REP=1 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "4096 or 8192" > gpurun_out/r2zo_tests.log 2>&1; echo rc=$? >> gpurun_out/r2zo_tests.log
