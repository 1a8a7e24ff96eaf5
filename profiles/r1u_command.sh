#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/v18_gputests.log 2>&1; echo rc=$? >> gpurun_out/v18_gputests.log
: > gpurun_out/v18.jsonl
run() { tag=$1; shift; line=$(timeout 400 env "$@" 2>>gpurun_out/v18.err | tail -1); python -c "import json,sys; d=json.loads(sys.argv[1]); d['run']=sys.argv[2]; print(json.dumps(d))" "$line" "$tag" >> gpurun_out/v18.jsonl || echo "{\"run\":\"$tag\",\"error\":1}" >> gpurun_out/v18.jsonl; }
for r in 1 2; do
for g in 32 0; do
run c4_g${g}_$r GCR_DRAIN_GROUP_MB=$g python bench.py --config C4 --mode incremental --dirty 0.01 --steps 6 --no-cpu-baseline
run c4_5_g${g}_$r GCR_DRAIN_GROUP_MB=$g python bench.py --config C4 --mode incremental --dirty 0.05 --steps 4 --no-cpu-baseline
done
done
run c2_g32 python bench.py --no-cpu-baseline --steps 10
run c2_g0 GCR_DRAIN_GROUP_MB=0 python bench.py --no-cpu-baseline --steps 10
GCR_TRACE=1 python bench.py --config C4 --mode incremental --dirty 0.01 --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2> gpurun_out/v18_trace.err
