#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stress.py tests/test_gpu_release.py tests/test_gpu_storage.py -x -q > gpurun_out/v7_tests.log 2>&1; echo rc=$? >> gpurun_out/v7_tests.log
: > gpurun_out/v7.jsonl
run() { tag=$1; shift; line=$(timeout 300 env "$@" 2>>gpurun_out/v7.err | tail -1); python -c "import json,sys; d=json.loads(sys.argv[1]); d['run']=sys.argv[2]; print(json.dumps(d))" "$line" "$tag" >> gpurun_out/v7.jsonl || echo "{\"run\":\"$tag\",\"error\":1}" >> gpurun_out/v7.jsonl; }
for sg in 1 0; do
run c2p4k_grp$sg GCR_SMALL_GROUPS=$sg python bench.py --no-cpu-baseline --steps 5 --page-size 4096
run c2p8k_grp$sg GCR_SMALL_GROUPS=$sg python bench.py --no-cpu-baseline --steps 5 --page-size 8192
run c5p4k_grp$sg GCR_SMALL_GROUPS=$sg python bench.py --config C5 --gib 16 --page-size 4096 --steps 3 --no-cpu-baseline
done
run c4p4k_grp1 python bench.py --config C4 --gib 16 --page-size 4096 --mode incremental --dirty 0.01 --steps 4 --no-cpu-baseline
