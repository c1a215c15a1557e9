# round-2 call W: warm Procrustes timelines (PTB_PROF) on configs 1-3, cfg1 launch list
mkdir -p gpurun_out
for c in 1 2 3; do
  PTB_PROF=1 timeout 600 python scripts/time_driver.py $c $c > gpurun_out/r02w_prof$c.log 2>&1
  echo "== cfg$c (second run, last iteration)"
  python - $c <<'PY'
import sys
lines=open(f'gpurun_out/r02w_prof{sys.argv[1]}.log').read().splitlines()
# second run's lines: after the first json line
idx=[i for i,l in enumerate(lines) if l.startswith('{')]
sec=lines[idx[0]+1:idx[1]]
# last update_svd block
starts=[i for i,l in enumerate(sec) if 'update: projections' in l]
blk=sec[starts[-1]:] if starts else sec[-30:]
print('\n'.join(blk[:40]))
print(lines[idx[1]][:400])
PY
done
python scripts/time_driver.py 1 > /dev/null 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02w_cfg1_launches.csv python scripts/time_driver.py 1 > /dev/null 2>&1; echo ncu=$?
python scripts/launch_table.py gpurun_out/r02w_cfg1_launches.csv 25
