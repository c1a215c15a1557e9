# round-2 session-5 call AJ: bench.py under torchrun with one rank (the N > 1 launch form, world 1)
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 1 --steps 2 --warmup 3 --no-sweep --no-cpu --no-pml --e2e-steps 1 > gpurun_out/r02dj_bench.json 2> gpurun_out/r02dj_bench.err; echo rc=$?
tail -c 700 gpurun_out/r02dj_bench.json; tail -3 gpurun_out/r02dj_bench.err
