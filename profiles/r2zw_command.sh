#!/bin/bash
# instance choice by page size: scan parity + C5 16 GiB at 256 KiB / 2 MiB and C2 at 64 KiB, hooks forced vs default
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2zw_smoke.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_verify.py -m gpu -q -x > gpurun_out/r2zw_tests.log 2>&1; echo rc=$? >> gpurun_out/r2zw_tests.log
for k in 1 2; do for H in 0 1; do
GCR_K1_HOOKS=$H timeout 600 python bench.py --no-cpu-baseline --sub-c4-gib 0 --config C5 --gib 16 --page-size 262144 --compress 0 --steps 3 > gpurun_out/r2zw_c5p256k_h${H}_$k.json 2>/dev/null
GCR_K1_HOOKS=$H timeout 600 python bench.py --no-cpu-baseline --sub-c4-gib 0 --config C5 --gib 16 --page-size 2097152 --compress 0 --steps 3 > gpurun_out/r2zw_c5p2m_h${H}_$k.json 2>/dev/null
GCR_K1_HOOKS=$H timeout 600 python bench.py --no-cpu-baseline --sub-c4-gib 0 --config C5 --gib 16 --compress 0 --steps 3 > gpurun_out/r2zw_c5p64k_h${H}_$k.json 2>/dev/null
done; done
