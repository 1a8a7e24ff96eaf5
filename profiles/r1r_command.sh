#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/v15_gputests.log 2>&1; echo rc=$? >> gpurun_out/v15_gputests.log
: > gpurun_out/v15.jsonl
run() { tag=$1; shift; line=$(timeout 400 env "$@" 2>>gpurun_out/v15.err | tail -1); python -c "import json,sys; d=json.loads(sys.argv[1]); d['run']=sys.argv[2]; print(json.dumps(d))" "$line" "$tag" >> gpurun_out/v15.jsonl || echo "{\"run\":\"$tag\",\"error\":1}" >> gpurun_out/v15.jsonl; }
run c4 python bench.py --config C4 --mode incremental --dirty 0.01 --steps 5 --no-cpu-baseline
run c4b python bench.py --config C4 --mode incremental --dirty 0.01 --steps 5 --no-cpu-baseline
run c4_5 python bench.py --config C4 --mode incremental --dirty 0.05 --steps 4 --no-cpu-baseline
run c2 python bench.py --no-cpu-baseline --steps 10
run c3 python bench.py --config C3 --no-cpu-baseline --steps 3
