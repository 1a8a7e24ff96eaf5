#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stress.py tests/test_gpu_release.py -x -q > gpurun_out/v2_new.log 2>&1; echo rc=$? >> gpurun_out/v2_new.log
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/v2_gputests.log 2>&1; echo rc=$? >> gpurun_out/v2_gputests.log
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/v2_c2.json 2> gpurun_out/v2_c2.err
timeout 300 python bench.py --no-cpu-baseline --release > gpurun_out/v2_c2_release.json 2> gpurun_out/v2_c2_release.err
for i in 1 2; do
timeout 300 python bench.py --config C4 --mode incremental --dirty 0.01 --steps 5 --chunk-mb 1024 --no-cpu-baseline > gpurun_out/v2_c4_$i.json 2>gpurun_out/v2_c4_$i.err
done
GCR_SCAN_PREFETCH=32768 timeout 300 python bench.py --config C4 --mode incremental --dirty 0.01 --steps 4 --chunk-mb 1024 --no-cpu-baseline > gpurun_out/v2_c4_pf32k.json 2>gpurun_out/v2_c4_pf32k.err
timeout 300 python bench.py --config C5 --gib 16 --page-size 4096 --steps 3 --chunk-mb 1024 --no-cpu-baseline > gpurun_out/v2_c5_4k.json 2>gpurun_out/v2_c5_4k.err
