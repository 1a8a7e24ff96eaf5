#!/bin/bash
# round 2: K6 over 64 KiB pieces (grid-stride over pieces, not descriptors);
# f4 decode descriptors written in place (host planning); tests + timings + benches
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2p_smoke.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_codec.py tests/test_gpu_parity.py tests/test_gpu_verify.py tests/test_gpu_stress.py -q -m gpu -x > gpurun_out/r2p_tests.log 2>&1; echo rc=$? >> gpurun_out/r2p_tests.log
timeout 300 python tools/restore_timing.py 4096 > gpurun_out/r2p_restore_timing_4k.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --sub-c4-gib 0 --compress 0 --direct-min-mb -1 --steps 5 > gpurun_out/r2p_bench_staged.json 2> gpurun_out/r2p_bench_staged.err
timeout 600 python bench.py --no-cpu-baseline --sub-c4-gib 0 --page-size 4096 --steps 5 > gpurun_out/r2p_bench_4k.json 2> gpurun_out/r2p_bench_4k.err
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r2p_bench.json 2> gpurun_out/r2p_bench.err
ncu --set full --clock-control none --import-source on -k regex:"k_scatter|k_zero_fill" -c 6 -o gpurun_out/r2p_k6k7 python bench.py --steps 1 --warmup 0 --no-cpu-baseline --sub-c4-gib 0 --compress 0 --direct-min-mb -1 > gpurun_out/r2p_ncu.log 2>&1
