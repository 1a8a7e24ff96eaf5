#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/v4_gputests.log 2>&1; echo rc=$? >> gpurun_out/v4_gputests.log
timeout 300 python bench.py > gpurun_out/v4_c2.json 2> gpurun_out/v4_c2.err
GCR_TRACE=1 timeout 300 python bench.py --config C4 --mode incremental --dirty 0.01 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/v4_c4_trace.json 2> gpurun_out/v4_c4_trace.err
timeout 600 python bench.py --config C3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/v4_c3.json 2> gpurun_out/v4_c3.err
