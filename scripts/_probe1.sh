set -x
nproc; free -g; lscpu | grep -i "model name\|socket\|thread\|core"; nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv
python -c "import torch;print(torch.cuda.mem_get_info())"
timeout 600 python bench.py --grid 4096 --batch 256 --steps 3 --warmup 3 --no-e2e --no-parareal --no-pml --no-sweep > gpurun_out/p1_bench4096.log 2>&1; echo rc=$?
tail -c 3000 gpurun_out/p1_bench4096.log
