#!/bin/bash
# round 2: codec tests (all), racecheck experiment (streaming vs coherent loads in
# the restore scatter), K8 per-warp stamps (where the fixed launch cost goes)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2e_build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_codec.py -q -m gpu > gpurun_out/r2e_codec_tests.log 2>&1; echo rc=$? >> gpurun_out/r2e_codec_tests.log
timeout 300 compute-sanitizer --tool racecheck python tools/racecheck_diag.py 65536 > gpurun_out/r2e_racecheck_nc.log 2>&1
GCR_DIAG_SCATTER_PLAIN=1 timeout 300 compute-sanitizer --tool racecheck python tools/racecheck_diag.py 65536 > gpurun_out/r2e_racecheck_plain.log 2>&1
timeout 300 compute-sanitizer --tool initcheck python tools/racecheck_diag.py 65536 > gpurun_out/r2e_initcheck.log 2>&1
GCR_SCAN_TIMES=1 timeout 300 python tools/scan_times.py 128 1024 4096 > gpurun_out/r2e_scan_times.log 2>&1
