#!/bin/bash
# D2H under SM load (does a concurrent HBM-streaming kernel slow the drain?);
# copy-kernel variant tests; default bench line
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2z_smoke.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/d2h_interference/d2h tools/d2h_interference/d2h_interference.cu
timeout 300 tools/d2h_interference/d2h > gpurun_out/r2z_d2h_interference.jsonl 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "variants or page_sizes" > gpurun_out/r2z_tests.log 2>&1; echo rc=$? >> gpurun_out/r2z_tests.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r2z_bench.json 2> gpurun_out/r2z_bench.err
GCR_TRACE=1 timeout 900 python bench.py --no-cpu-baseline --sub-c4-gib 0 --steps 3 > gpurun_out/r2z_bench_trace.json 2> gpurun_out/r2z_bench_trace.err
