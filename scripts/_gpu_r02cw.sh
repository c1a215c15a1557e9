# round-2 session-5 call W: ncu --set full of the headline kernel under the two-lane plan (4096^2, 32-slice launch)
python scripts/prof_prop.py 4096 64 1 > gpurun_out/r02cw_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_wave2 -s 8 -c 1 -f -o gpurun_out/r02cw_k1 python scripts/prof_prop.py 4096 64 1 > gpurun_out/r02cw_ncu.log 2>&1; echo ncu=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02cw_launches.csv python scripts/prof_prop.py 4096 64 1 > /dev/null 2>&1; echo launches=$?
tail -2 gpurun_out/r02cw_plain.log
