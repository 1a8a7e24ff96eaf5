#!/bin/bash
# speculative prefix H2D in the f4 restore (issued before host validation):
# restore-path tests, restore timeline, default bench line; C4 1 % with and
# without the ramped chunk plan (same box, alternating)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2w_smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x tests/test_gpu_codec.py tests/test_gpu_verify.py tests/test_gpu_release.py tests/test_gpu_storage.py tests/test_gpu_abi.py > gpurun_out/r2w_tests.log 2>&1; echo rc=$? >> gpurun_out/r2w_tests.log
GCR_TRACE=1 timeout 300 python tools/restore_timing.py 65536 > gpurun_out/r2w_rt.log 2> gpurun_out/r2w_rt.err
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r2w_bench.json 2> gpurun_out/r2w_bench.err
for k in 1 2; do for R in 0 1; do
GCR_CHUNK_RAMP=$R timeout 600 python bench.py --no-cpu-baseline --sub-c4-gib 0 --config C4 --mode incremental --dirty 0.01 --steps 5 --compress 0 > gpurun_out/r2w_c4_ramp${R}_$k.json 2> gpurun_out/r2w_c4_ramp${R}_$k.err
done; done
