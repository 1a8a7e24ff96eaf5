#!/bin/bash
# Measurement sweep over BASELINE.json's configs (run on the GPU box via gpurun).
# One JSON line per run is appended to gpurun_out/sweep.jsonl, tagged with "run".
# Round 2: the f4 codec is bench.py's default (--compress 1); uncompressed runs
# say --compress 0.  The C4-shaped sub-record of the default line is off here.
set -u
OUT=gpurun_out/sweep.jsonl
mkdir -p gpurun_out
: > $OUT
run() {  # tag, args...
  tag=$1; shift
  line=$(timeout 900 python bench.py --no-cpu-baseline --sub-c4-gib 0 "$@" 2> gpurun_out/sweep_$tag.err | tail -1)
  python -c "import json,sys; d=json.loads(sys.argv[1]); d['run']=sys.argv[2]; print(json.dumps(d))" "$line" "$tag" >> $OUT \
    || echo "{\"run\": \"$tag\", \"error\": \"$(tail -1 gpurun_out/sweep_$tag.err | tr -d '\"')\"}" >> $OUT
}
run C1 --config C1 --steps 10
run C2 --config C2 --steps 10
run C2_plain --config C2 --steps 10 --compress 0
run C2_P4K --config C2 --page-size 4096 --steps 5
run C2_P2M --config C2 --page-size 2097152 --steps 5
run C3 --config C3 --steps 3 --warmup 3
run C3_plain --config C3 --steps 3 --warmup 3 --compress 0
run C4_inc1 --config C4 --mode incremental --dirty 0.01 --steps 5 --compress 0
run C4_inc5 --config C4 --mode incremental --dirty 0.05 --steps 5 --compress 0
run C4_inc1_f1 --config C4 --mode incremental --dirty 0.01 --steps 5 --compress 0 --in-scan-pack 1
run C5_16G_P4K --config C5 --gib 16 --page-size 4096 --steps 3 --compress 0
run C5_16G_P64K --config C5 --gib 16 --steps 3 --compress 0
run C5_16G_P2M --config C5 --gib 16 --page-size 2097152 --steps 3 --compress 0
run C5_64G_P64K --config C5 --gib 64 --steps 3 --warmup 3 --compress 0
run C2_release --config C2 --steps 5 --release
mkdir -p /tmp/gcr_sweep_store
run C2_storage --config C2 --steps 3 --warmup 1 --storage /tmp/gcr_sweep_store
rm -rf /tmp/gcr_sweep_store
echo done
