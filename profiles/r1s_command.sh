#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/v16.jsonl
run() { tag=$1; shift; line=$(timeout 400 env "$@" 2>>gpurun_out/v16.err | tail -1); python -c "import json,sys; d=json.loads(sys.argv[1]); d['run']=sys.argv[2]; print(json.dumps(d))" "$line" "$tag" >> gpurun_out/v16.jsonl || echo "{\"run\":\"$tag\",\"error\":1}" >> gpurun_out/v16.jsonl; }
for r in 1 2; do
for ramp in 1 0; do
run c4_ramp${ramp}_$r GCR_CHUNK_RAMP=$ramp python bench.py --config C4 --mode incremental --dirty 0.01 --steps 6 --no-cpu-baseline
run c4_5_ramp${ramp}_$r GCR_CHUNK_RAMP=$ramp python bench.py --config C4 --mode incremental --dirty 0.05 --steps 4 --no-cpu-baseline
done
done
GCR_TRACE=1 python bench.py --config C4 --mode incremental --dirty 0.01 --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2> gpurun_out/v16_trace_ramp1.err
GCR_CHUNK_RAMP=0 GCR_TRACE=1 python bench.py --config C4 --mode incremental --dirty 0.01 --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2> gpurun_out/v16_trace_ramp0.err
