#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_storage.py tests/test_gpu_stress.py tests/test_gpu_release.py -x -q > gpurun_out/v3_tests.log 2>&1; echo rc=$? >> gpurun_out/v3_tests.log
(df -h /tmp /root /dev/shm; lsblk; nproc; free -g) > gpurun_out/v3_sys.txt 2>&1
: > gpurun_out/v3.jsonl
run() { tag=$1; shift; line=$(timeout 300 env "$@" 2>>gpurun_out/v3.err | tail -1); python -c "import json,sys; d=json.loads(sys.argv[1]); d['run']=sys.argv[2]; print(json.dumps(d))" "$line" "$tag" >> gpurun_out/v3.jsonl || echo "{\"run\":\"$tag\",\"error\":1}" >> gpurun_out/v3.jsonl; }
for f in 10 6 4; do
run c4_free$f GCR_FREE_SMS=$f python bench.py --config C4 --mode incremental --dirty 0.01 --steps 5 --chunk-mb 1024 --no-cpu-baseline
done
run c2_free4 GCR_FREE_SMS=4 python bench.py --no-cpu-baseline --steps 5
run c2_chunk1g python bench.py --no-cpu-baseline --steps 5 --chunk-mb 1024
mkdir -p /tmp/gcrstore
run c2_storage python bench.py --no-cpu-baseline --steps 3 --warmup 1 --storage /tmp/gcrstore
rm -rf /tmp/gcrstore
