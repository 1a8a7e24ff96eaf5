#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/v8_smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/v8_gputests.log 2>&1; echo rc=$? >> gpurun_out/v8_gputests.log
timeout 400 python bench.py > gpurun_out/v8_bench.json 2> gpurun_out/v8_bench.err
timeout 300 python bench.py --impl reference --steps 2 --warmup 0 > gpurun_out/v8_bench_ref.json 2> gpurun_out/v8_bench_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 1000 --csv --log-file gpurun_out/r1m_launches_bench.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r1m_launch_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_scan -c 2 -o gpurun_out/r1m_kscan python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/r1m_ncu_kscan.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_scan_grp -c 2 -o gpurun_out/r1m_kscan_grp python bench.py --steps 1 --warmup 0 --no-cpu-baseline --page-size 4096 > gpurun_out/r1m_ncu_kscan_grp.log 2>&1
