mkdir -p gpurun_out
( nproc; lscpu | grep -E "Model name|Socket|Thread|Core|NUMA node\(s\)"; free -g; nvidia-smi --query-gpu=name,clocks.max.sm,memory.total --format=csv; nvidia-smi topo -m ) > gpurun_out/box_info.txt 2>&1
nvcc -O2 -gencode arch=compute_100a,code=sm_100a tools/probe_mc.cu -o /tmp/probe_mc -lcuda && timeout 60 /tmp/probe_mc > gpurun_out/probe_mc.txt 2>&1; cat gpurun_out/probe_mc.txt
bash tools/gpu_sanitize.sh
NO_BENCH=1 TAG=r2a bash tools/gpu_round.sh
