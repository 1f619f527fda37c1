nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc; lscpu | grep -E "Model name|^CPU\(s\)|Socket|Thread"
./tools/microbench/fp32_pipe
