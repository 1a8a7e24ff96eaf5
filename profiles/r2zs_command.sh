#!/bin/bash
# final evidence after the hook-free K1 instance: smoke,
# every GPU test, default bench (with cpu_baseline), reference arm, 2 ranks,
# the launch list, ncu of k_scan (exact name) and the C3 / C5 lines
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2zs_smoke.log 2>&1
timeout 2700 python -m pytest tests -m gpu -q > gpurun_out/r2zs_gputests.log 2>&1; echo rc=$? >> gpurun_out/r2zs_gputests.log
timeout 900 python bench.py > gpurun_out/r2zs_bench.json 2> gpurun_out/r2zs_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/r2zs_bench_ref.json 2> gpurun_out/r2zs_bench_ref.err
timeout 600 python bench.py --gpus 2 --steps 5 --no-cpu-baseline --sub-c4-gib 0 > gpurun_out/r2zs_bench_2ranks.json 2> gpurun_out/r2zs_bench_2ranks.err
timeout 900 python bench.py --no-cpu-baseline --sub-c4-gib 0 --config C3 --steps 3 > gpurun_out/r2zs_c3.json 2>/dev/null
timeout 900 python bench.py --no-cpu-baseline --sub-c4-gib 0 --config C5 --gib 64 --steps 3 --compress 0 > gpurun_out/r2zs_c5_64g.json 2>/dev/null
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r2zs_launches_bench.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --sub-c4-gib 0 > gpurun_out/r2zs_launch_bench.log 2>&1
NCU="ncu --set full --clock-control none --import-source on"
$NCU -k regex:"k_scan<" -c 2 -o gpurun_out/r2zs_kscan python bench.py --steps 1 --warmup 0 --no-cpu-baseline --sub-c4-gib 0 > gpurun_out/r2zs_ncu1.log 2>&1
