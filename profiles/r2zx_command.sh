#!/bin/bash
# FINAL: every GPU test, smoke, the default bench line, the reference arm, 2 ranks
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2zx_smoke.log 2>&1
timeout 2700 python -m pytest tests -m gpu -q > gpurun_out/r2zx_gputests.log 2>&1; echo rc=$? >> gpurun_out/r2zx_gputests.log
timeout 900 python bench.py > gpurun_out/r2zx_bench.json 2> gpurun_out/r2zx_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/r2zx_bench_ref.json 2> gpurun_out/r2zx_bench_ref.err
timeout 600 python bench.py --gpus 2 --steps 5 --no-cpu-baseline --sub-c4-gib 0 > gpurun_out/r2zx_bench_2ranks.json 2> gpurun_out/r2zx_bench_2ranks.err
