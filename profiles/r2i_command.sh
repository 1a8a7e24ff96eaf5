#!/bin/bash
# round 2: f1 diagnostics with a 2 s bound on the in-kernel waits
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2i_build.log 2>&1
export GCR_ISP_WAIT_MS=2000
timeout 600 python -m pytest tests/test_gpu_inscan.py -q -m gpu -x > gpurun_out/r2i_inscan.log 2>&1; echo rc=$? >> gpurun_out/r2i_inscan.log
timeout 300 python bench.py --no-cpu-baseline --config C4 --gib 4 --mode incremental --dirty 0.01 --steps 3 --compress 0 --in-scan-pack 1 > gpurun_out/r2i_c4g4.json 2> gpurun_out/r2i_c4g4.err
