#!/bin/bash
# round 2: K6 TMA scatter without descriptor walks; parity; staged-restore bench;
# the config sweep (tools/sweep.sh) on the current code
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2n_smoke.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stress.py tests/test_gpu_release.py -q -m gpu -x > gpurun_out/r2n_tests.log 2>&1; echo rc=$? >> gpurun_out/r2n_tests.log
timeout 600 python bench.py --no-cpu-baseline --sub-c4-gib 0 --compress 0 --direct-min-mb -1 --steps 5 > gpurun_out/r2n_bench_staged.json 2> gpurun_out/r2n_bench_staged.err
bash tools/sweep.sh > gpurun_out/r2n_sweep_stdout.txt 2>&1
cp gpurun_out/sweep.jsonl gpurun_out/r2n_sweep.jsonl
