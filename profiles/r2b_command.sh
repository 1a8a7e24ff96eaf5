#!/bin/bash
# round 2: new verify-failure tests, ABI semantics (unwatched lock, checkpoint_abort,
# RELEASED after a failed restore), then the full-size bit-exact parity tests
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2b_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_verify.py tests/test_gpu_abi.py tests/test_gpu_release.py -q -m gpu > gpurun_out/r2b_new.log 2>&1; echo rc=$? >> gpurun_out/r2b_new.log
( time timeout 2400 python -m pytest tests/test_gpu_fullsize.py -q -m gpu --durations=10 ) > gpurun_out/r2b_fullsize.log 2>&1; echo rc=$? >> gpurun_out/r2b_fullsize.log
