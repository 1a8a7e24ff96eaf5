#!/bin/bash
mkdir -p gpurun_out
GCR_BATCH_MIN=65536 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stress.py -x -q > gpurun_out/v5_tests_batch.log 2>&1; echo rc=$? >> gpurun_out/v5_tests_batch.log
: > gpurun_out/v5.jsonl
run() { tag=$1; shift; line=$(timeout 300 env "$@" 2>>gpurun_out/v5.err | tail -1); python -c "import json,sys; d=json.loads(sys.argv[1]); d['run']=sys.argv[2]; print(json.dumps(d))" "$line" "$tag" >> gpurun_out/v5.jsonl || echo "{\"run\":\"$tag\",\"error\":1}" >> gpurun_out/v5.jsonl; }
run c4_base GCR_TRACE=1 python bench.py --config C4 --mode incremental --dirty 0.01 --steps 5 --no-cpu-baseline
run c4_batch64k GCR_TRACE=1 GCR_BATCH_MIN=65536 python bench.py --config C4 --mode incremental --dirty 0.01 --steps 5 --no-cpu-baseline
run c4_5_base python bench.py --config C4 --mode incremental --dirty 0.05 --steps 4 --no-cpu-baseline
run c4_5_batch64k GCR_BATCH_MIN=65536 python bench.py --config C4 --mode incremental --dirty 0.05 --steps 4 --no-cpu-baseline
run c2_batch64k GCR_BATCH_MIN=65536 python bench.py --no-cpu-baseline --steps 5
run c2_batch4k GCR_BATCH_MIN=4096 python bench.py --no-cpu-baseline --steps 5
