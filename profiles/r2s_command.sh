#!/bin/bash
# K1g full-group fast path (c8dae84): same-box scan A/B against 8671537, the
# 4/8 KiB parity + verify tests on the new code, and C2 at 4K/64K/2M pages
mkdir -p gpurun_out
timeout 600 python tools/scan_ab.py 1024 4096 > gpurun_out/r2s_scan_ab.log 2>&1
timeout 1200 python -m pytest -q -m gpu tests/test_gpu_parity.py tests/test_gpu_verify.py -k "4096 or 8192 or grp or K1g" > gpurun_out/r2s_tests.log 2>&1; echo rc=$? >> gpurun_out/r2s_tests.log
for P in 4096 65536 2097152; do
  timeout 600 python bench.py --no-cpu-baseline --sub-c4-gib 0 --config C2 --page-size $P --steps 5 --compress 0 > gpurun_out/r2s_c2_p$P.json 2> gpurun_out/r2s_c2_p$P.err
done
timeout 600 python bench.py --no-cpu-baseline --sub-c4-gib 0 --config C4 --mode incremental --dirty 0.01 --steps 5 --compress 0 > gpurun_out/r2s_c4_inc1.json 2> gpurun_out/r2s_c4_inc1.err
