#!/bin/bash
# round 2: staged-group fix; f4 checkpoint sub-chunk trace; tests; benches
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2q_smoke.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stress.py tests/test_gpu_codec.py -q -m gpu -x > gpurun_out/r2q_tests.log 2>&1; echo rc=$? >> gpurun_out/r2q_tests.log
timeout 600 python bench.py --no-cpu-baseline --sub-c4-gib 0 --compress 0 --direct-min-mb -1 --steps 5 > gpurun_out/r2q_bench_staged.json 2> gpurun_out/r2q_bench_staged.err
GCR_TRACE=1 timeout 600 python bench.py --no-cpu-baseline --sub-c4-gib 0 --steps 2 --warmup 1 > gpurun_out/r2q_bench_trace.json 2> gpurun_out/r2q_bench_trace.err
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r2q_bench.json 2> gpurun_out/r2q_bench.err
