# round-2 call Z: PML frame mode (interior k_wave2 + band tiles) parity + timing
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pml.py -q -x -rf 2>&1 | tail -3
python scripts/time_pml.py 2>&1 | tail -4
PTB_PML_FRAME=0 python scripts/time_pml.py 2>&1 | tail -4
timeout 1500 python bench.py --no-sweep --no-parareal --no-cpu --no-e2e --steps 3 > gpurun_out/r02z_bench.json 2> gpurun_out/r02z_bench.err; echo bench_rc=$?
python -c "
import json;d=json.loads(open('gpurun_out/r02z_bench.json').read().splitlines()[-1]);print(json.dumps(d.get('cfg4_pml')))"
