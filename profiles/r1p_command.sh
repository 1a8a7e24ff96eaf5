#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stress.py tests/test_gpu_abi.py -x -q > gpurun_out/v13_tests.log 2>&1; echo rc=$? >> gpurun_out/v13_tests.log
: > gpurun_out/v13.jsonl
run() { tag=$1; shift; line=$(timeout 400 env "$@" 2>>gpurun_out/v13.err | tail -1); python -c "import json,sys; d=json.loads(sys.argv[1]); d['run']=sys.argv[2]; print(json.dumps(d))" "$line" "$tag" >> gpurun_out/v13.jsonl || echo "{\"run\":\"$tag\",\"error\":1}" >> gpurun_out/v13.jsonl; }
run c2 python bench.py --no-cpu-baseline --steps 10
run c3 python bench.py --config C3 --no-cpu-baseline --steps 3
run c4 python bench.py --config C4 --mode incremental --dirty 0.01 --steps 5 --no-cpu-baseline
run c5p4k python bench.py --config C5 --gib 16 --page-size 4096 --steps 3 --no-cpu-baseline
run c2b python bench.py --no-cpu-baseline --steps 10
