#!/bin/bash
# K1 / K8 instance without the f1 hooks (k_scan<false>) for every launch that
# does not use the in-scan pack: parity (parity, in-scan, verify, fuzz, stress),
# same-box A/B against the hooked instance (GCR_K1_HOOKS=1) on C4 1 % and C2
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2zr_smoke.log 2>&1
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_inscan.py tests/test_gpu_verify.py tests/test_gpu_fuzz.py tests/test_gpu_stress.py -m gpu -q -x > gpurun_out/r2zr_tests.log 2>&1; echo rc=$? >> gpurun_out/r2zr_tests.log
for k in 1 2 3; do for H in 0 1; do
GCR_K1_HOOKS=$H timeout 600 python bench.py --no-cpu-baseline --sub-c4-gib 0 --config C4 --mode incremental --dirty 0.01 --steps 5 --compress 0 > gpurun_out/r2zr_c4_h${H}_$k.json 2>/dev/null
GCR_K1_HOOKS=$H timeout 600 python bench.py --no-cpu-baseline --sub-c4-gib 0 --steps 10 > gpurun_out/r2zr_c2_h${H}_$k.json 2>/dev/null
done; done
