#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/v11_gputests.log 2>&1; echo rc=$? >> gpurun_out/v11_gputests.log
: > gpurun_out/v11.jsonl
run() { tag=$1; shift; line=$(timeout 300 env "$@" 2>>gpurun_out/v11.err | tail -1); python -c "import json,sys; d=json.loads(sys.argv[1]); d['run']=sys.argv[2]; print(json.dumps(d))" "$line" "$tag" >> gpurun_out/v11.jsonl || echo "{\"run\":\"$tag\",\"error\":1}" >> gpurun_out/v11.jsonl; }
run c2 python bench.py --no-cpu-baseline --steps 10
run c4 python bench.py --config C4 --mode incremental --dirty 0.01 --steps 5 --no-cpu-baseline
run c2p2m python bench.py --no-cpu-baseline --steps 5 --page-size 2097152
GCR_SCAN_TIMES=1 python scratch/scan_size.py > gpurun_out/v11_scan_size.jsonl 2> gpurun_out/v11_scan_times.err
