mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2a_smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2a_gputests.log 2>&1; echo rc=$? >> gpurun_out/r2a_gputests.log
timeout 400 python bench.py > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err
nproc > gpurun_out/r2a_host.txt; lscpu >> gpurun_out/r2a_host.txt; nvidia-smi topo -m >> gpurun_out/r2a_host.txt 2>&1; free -g >> gpurun_out/r2a_host.txt; numactl -H >> gpurun_out/r2a_host.txt 2>&1; cat /sys/bus/pci/devices/*/numa_node 2>/dev/null | sort | uniq -c >> gpurun_out/r2a_host.txt; nvidia-smi -q | grep -i -A3 "bus id" | head >> gpurun_out/r2a_host.txt
