#!/bin/bash
# K4 TMA with interleaved item assignment: parity tests for K4/K6, same-box
# A/B (TMA vs vector) on the all-staged C2 round trip and C4 1 %; host
# overhead breakdown of the incremental step; ncu of k_pack_tma
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2y_smoke.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stress.py tests/test_gpu_inscan.py -m gpu -q -x > gpurun_out/r2y_tests.log 2>&1; echo rc=$? >> gpurun_out/r2y_tests.log
for k in 1 2; do for T in 1 0; do
GCR_TMA_COPY=$T timeout 600 python bench.py --no-cpu-baseline --sub-c4-gib 0 --compress 0 --direct-min-mb -1 --steps 5 > gpurun_out/r2y_staged_tma${T}_$k.json 2> /dev/null
GCR_TMA_COPY=$T timeout 600 python bench.py --no-cpu-baseline --sub-c4-gib 0 --config C4 --mode incremental --dirty 0.01 --steps 5 --compress 0 > gpurun_out/r2y_c4_tma${T}_$k.json 2> /dev/null
done; done
timeout 300 python tools/host_overhead.py 8 8 > gpurun_out/r2y_host_overhead_8g.log 2>&1
timeout 600 python tools/host_overhead.py 40 6 > gpurun_out/r2y_host_overhead_40g.log 2>&1
NCU="ncu --set full --clock-control none --import-source on"
timeout 900 $NCU -k regex:"k_pack" -c 4 -o gpurun_out/r2y_pack python bench.py --steps 1 --warmup 0 --no-cpu-baseline --sub-c4-gib 0 --compress 0 --direct-min-mb -1 > gpurun_out/r2y_ncu.log 2>&1
