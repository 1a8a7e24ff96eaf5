#!/bin/bash
# restore region ring (H2Ds no longer wait for the decode two groups back):
# restore-path GPU tests, the default bench line, restore timing; plus the
# C4-shaped 8 GiB sub-record with and without the ramped chunk plan
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2u_smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x tests/test_gpu_codec.py tests/test_gpu_parity.py tests/test_gpu_verify.py tests/test_gpu_release.py tests/test_gpu_storage.py > gpurun_out/r2u_tests.log 2>&1; echo rc=$? >> gpurun_out/r2u_tests.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r2u_bench.json 2> gpurun_out/r2u_bench.err
timeout 300 python tools/restore_timing.py 65536 > gpurun_out/r2u_restore_timing.log 2>&1
for R in 0 1; do
GCR_CHUNK_RAMP=$R timeout 600 python bench.py --no-cpu-baseline --sub-c4-gib 0 --config C4 --gib 8 --mode incremental --dirty 0.01 --steps 10 --compress 0 > gpurun_out/r2u_c4g8_ramp$R.json 2> gpurun_out/r2u_c4g8_ramp$R.err
done
