#!/bin/bash
# round 2: same-box A/B of the scan kernel vs round 1's (tools/scan_ab.py),
# tests after moving the f1 state to shared memory, TMA K6 (staged restore),
# compressed sub-chunks (default bench line)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2m_smoke.log 2>&1
timeout 600 python tools/scan_ab.py 1024 4096 > gpurun_out/r2m_scan_ab.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_inscan.py tests/test_gpu_codec.py tests/test_gpu_parity.py tests/test_gpu_verify.py -q -m gpu -x > gpurun_out/r2m_tests.log 2>&1; echo rc=$? >> gpurun_out/r2m_tests.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r2m_bench.json 2> gpurun_out/r2m_bench.err
timeout 600 python bench.py --no-cpu-baseline --sub-c4-gib 0 --compress 0 --direct-min-mb -1 --steps 5 > gpurun_out/r2m_bench_staged.json 2> gpurun_out/r2m_bench_staged.err
timeout 600 python tools/scan_ab.py 1024 > gpurun_out/r2m_scan_ab2.log 2>&1
