#!/bin/bash
# K1 full-mode tail merge (chunks 1.. as one range, published together):
# parity (parity/fuzz/codec/stress), same-box A/B GCR_SCAN_MERGE=0/1 on C3,
# C5 16 GiB (64K, 4K) and C2 at 4 KiB pages (K1g; C2 has 2 chunks: no merge)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2zk_smoke.log 2>&1
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_codec.py tests/test_gpu_stress.py tests/test_gpu_verify.py -m gpu -q -x > gpurun_out/r2zk_tests.log 2>&1; echo rc=$? >> gpurun_out/r2zk_tests.log
for k in 1 2; do for M in 1 0; do
GCR_SCAN_MERGE=$M timeout 900 python bench.py --no-cpu-baseline --sub-c4-gib 0 --config C3 --steps 3 > gpurun_out/r2zk_c3_m${M}_$k.json 2>/dev/null
GCR_SCAN_MERGE=$M timeout 900 python bench.py --no-cpu-baseline --sub-c4-gib 0 --config C5 --gib 16 --steps 3 --compress 0 > gpurun_out/r2zk_c5_m${M}_$k.json 2>/dev/null
GCR_SCAN_MERGE=$M timeout 900 python bench.py --no-cpu-baseline --sub-c4-gib 0 --config C5 --gib 16 --page-size 4096 --steps 3 --compress 0 > gpurun_out/r2zk_c5p4k_m${M}_$k.json 2>/dev/null
done; done
