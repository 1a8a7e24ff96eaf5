#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/v10.jsonl
run() { tag=$1; shift; line=$(timeout 300 env "$@" 2>>gpurun_out/v10.err | tail -1); python -c "import json,sys; d=json.loads(sys.argv[1]); d['run']=sys.argv[2]; print(json.dumps(d))" "$line" "$tag" >> gpurun_out/v10.jsonl || echo "{\"run\":\"$tag\",\"error\":1}" >> gpurun_out/v10.jsonl; }
run p4k_pfb0 GCR_GRP_PF_BLOCK=0 python bench.py --no-cpu-baseline --steps 5 --page-size 4096
run p4k_pfb4 GCR_GRP_PF_BLOCK=4 python bench.py --no-cpu-baseline --steps 5 --page-size 4096
run p4k_pfb6 GCR_GRP_PF_BLOCK=6 python bench.py --no-cpu-baseline --steps 5 --page-size 4096
run p4k_pfoff GCR_SCAN_PREFETCH=0 python bench.py --no-cpu-baseline --steps 5 --page-size 4096
run c5p4k_pfb0 GCR_GRP_PF_BLOCK=0 python bench.py --config C5 --gib 16 --page-size 4096 --steps 3 --no-cpu-baseline
run c5p4k_pfb4 GCR_GRP_PF_BLOCK=4 python bench.py --config C5 --gib 16 --page-size 4096 --steps 3 --no-cpu-baseline
run c5p4k_pfoff GCR_SCAN_PREFETCH=0 python bench.py --config C5 --gib 16 --page-size 4096 --steps 3 --no-cpu-baseline
ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none -k regex:k_scan -c 4 --csv --log-file gpurun_out/v10_ncu_pfb4.csv env GCR_GRP_PF_BLOCK=4 python bench.py --steps 1 --warmup 0 --no-cpu-baseline --page-size 4096 > /dev/null 2>&1
ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none -k regex:k_scan -c 4 --csv --log-file gpurun_out/v10_ncu_pfoff.csv env GCR_SCAN_PREFETCH=0 python bench.py --steps 1 --warmup 0 --no-cpu-baseline --page-size 4096 > /dev/null 2>&1
