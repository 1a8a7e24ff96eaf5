#!/bin/bash
# final round-1 evidence: smoke, every GPU test, the default bench line (+cpu_baseline),
# the reference arm, the ncu launch list and full captures, then the config sweep
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/v14_smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/v14_gputests.log 2>&1; echo rc=$? >> gpurun_out/v14_gputests.log
timeout 400 python bench.py > gpurun_out/v14_bench.json 2> gpurun_out/v14_bench.err
timeout 300 python bench.py --impl reference --steps 2 --warmup 0 > gpurun_out/v14_bench_ref.json 2> gpurun_out/v14_bench_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 1000 --csv --log-file gpurun_out/r1q_launches_bench.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r1q_launch_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_scan -c 2 -o gpurun_out/r1q_kscan python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/r1q_ncu_kscan.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_scan_grp -c 2 -o gpurun_out/r1q_kscan_grp python bench.py --steps 1 --warmup 0 --no-cpu-baseline --page-size 4096 > gpurun_out/r1q_ncu_kscan_grp.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_pack|k_scatter|k_zero|k_tile_scan|k_pm" -c 8 -o gpurun_out/r1q_kother python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/r1q_ncu_kother.log 2>&1
bash tools/sweep.sh > gpurun_out/sweep_stdout.txt 2>&1
