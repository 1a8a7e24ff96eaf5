#!/bin/bash
# TMA bulk-copy ring for K4 pack / K6 scatter (default; GCR_TMA_COPY=0 = vector
# copies) + the restore's fence moved ahead of the speculative prefix H2D:
# all GPU tests, smoke, default bench, restore timing, same-box A/B of the
# all-staged C2 round trip and C4 1 %, ncu of the TMA kernels
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2x_smoke.log 2>&1
timeout 2000 python -m pytest tests -m gpu -q -x > gpurun_out/r2x_gputests.log 2>&1; echo rc=$? >> gpurun_out/r2x_gputests.log
GCR_TRACE=1 timeout 300 python tools/restore_timing.py 65536 > gpurun_out/r2x_rt.log 2> gpurun_out/r2x_rt.err
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r2x_bench.json 2> gpurun_out/r2x_bench.err
for k in 1 2; do for T in 1 0; do
GCR_TMA_COPY=$T timeout 600 python bench.py --no-cpu-baseline --sub-c4-gib 0 --compress 0 --direct-min-mb -1 --steps 5 > gpurun_out/r2x_staged_tma${T}_$k.json 2> /dev/null
GCR_TMA_COPY=$T timeout 600 python bench.py --no-cpu-baseline --sub-c4-gib 0 --config C4 --mode incremental --dirty 0.01 --steps 5 --compress 0 > gpurun_out/r2x_c4_tma${T}_$k.json 2> /dev/null
done; done
NCU="ncu --set full --clock-control none --import-source on"
timeout 900 $NCU -k regex:"k_scatter|k_pack" -c 6 -o gpurun_out/r2x_tma python bench.py --steps 1 --warmup 0 --no-cpu-baseline --sub-c4-gib 0 --compress 0 --direct-min-mb -1 > gpurun_out/r2x_ncu.log 2>&1
