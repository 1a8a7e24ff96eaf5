#!/bin/bash
# round 2: conflict-free table staging; K8 stamps with per-SM exit means; bench
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2g_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_verify.py -q -m gpu -x > gpurun_out/r2g_tests.log 2>&1; echo rc=$? >> gpurun_out/r2g_tests.log
GCR_SCAN_TIMES=1 timeout 300 python tools/scan_times.py 128 1024 4096 > gpurun_out/r2g_scan_times.log 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r2g_bench.json 2> gpurun_out/r2g_bench.err
timeout 600 python bench.py --no-cpu-baseline --page-size 4096 > gpurun_out/r2g_bench_4k.json 2> gpurun_out/r2g_bench_4k.err
timeout 600 python bench.py --no-cpu-baseline --page-size 2097152 > gpurun_out/r2g_bench_2m.json 2> gpurun_out/r2g_bench_2m.err
