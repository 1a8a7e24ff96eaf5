#!/bin/bash
# FINAL evidence on the final code (hook-free K1 / K1g instances): smoke, every
# GPU test, the default bench line, reference arm, 2 ranks, the config sweep
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2zu_smoke.log 2>&1
timeout 2700 python -m pytest tests -m gpu -q > gpurun_out/r2zu_gputests.log 2>&1; echo rc=$? >> gpurun_out/r2zu_gputests.log
timeout 900 python bench.py > gpurun_out/r2zu_bench.json 2> gpurun_out/r2zu_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/r2zu_bench_ref.json 2> gpurun_out/r2zu_bench_ref.err
timeout 600 python bench.py --gpus 2 --steps 5 --no-cpu-baseline --sub-c4-gib 0 > gpurun_out/r2zu_bench_2ranks.json 2> gpurun_out/r2zu_bench_2ranks.err
bash tools/sweep.sh > gpurun_out/r2zu_sweep_stdout.txt 2>&1
cp gpurun_out/sweep.jsonl gpurun_out/r2zu_sweep.jsonl
