#!/bin/bash
# ramp-down-only chunk plan (GCR_CHUNK_RAMP=2): parity, same-box A/B against
# uniform chunks (0) and the two-ended ramp (1) on C4 1 % at 40 GiB and on the
# 8 GiB shape of the default line's sub-record
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2ze_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k ramp > gpurun_out/r2ze_tests.log 2>&1; echo rc=$? >> gpurun_out/r2ze_tests.log
for k in 1 2; do for R in 0 2 1; do
GCR_CHUNK_RAMP=$R timeout 600 python bench.py --no-cpu-baseline --sub-c4-gib 0 --config C4 --mode incremental --dirty 0.01 --steps 5 --compress 0 > gpurun_out/r2ze_c4_ramp${R}_$k.json 2>/dev/null
GCR_CHUNK_RAMP=$R timeout 600 python bench.py --no-cpu-baseline --sub-c4-gib 0 --config C4 --gib 8 --mode incremental --dirty 0.01 --steps 10 --compress 0 > gpurun_out/r2ze_c4g8_ramp${R}_$k.json 2>/dev/null
done; done
