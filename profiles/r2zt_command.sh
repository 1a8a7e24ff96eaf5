#!/bin/bash
# K1g hook-free immediate-base instance (dynamic smem base 0x400, probe-verified):
# probe log, K1g parity / verify / in-scan / fuzz tests, same-box A/B against
# the hooked instance (GCR_K1_HOOKS=1) at 4 KiB pages (C2, C5 16 GiB)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2zt_smoke.log 2>&1
GCR_TRACE=1 python -c "
import torch; from paper_2502_16631_b200 import gcr; c=gcr.Context(0); c.close()" > gpurun_out/r2zt_probe.log 2>&1
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_verify.py tests/test_gpu_inscan.py tests/test_gpu_fuzz.py tests/test_gpu_codec.py -m gpu -q -x > gpurun_out/r2zt_tests.log 2>&1; echo rc=$? >> gpurun_out/r2zt_tests.log
for k in 1 2; do for H in 0 1; do
GCR_K1_HOOKS=$H timeout 600 python bench.py --no-cpu-baseline --sub-c4-gib 0 --page-size 4096 --compress 0 --steps 5 > gpurun_out/r2zt_c2p4k_h${H}_$k.json 2>/dev/null
GCR_K1_HOOKS=$H timeout 600 python bench.py --no-cpu-baseline --sub-c4-gib 0 --config C5 --gib 16 --page-size 4096 --compress 0 --steps 3 > gpurun_out/r2zt_c5p4k_h${H}_$k.json 2>/dev/null
done; done
