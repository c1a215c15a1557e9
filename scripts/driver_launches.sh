# per-kernel launch list of the device parareal driver on one config (ncu, 1 metric, cold & serialised)
# usage: bash scripts/driver_launches.sh CFG[:K] OUT_CSV
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$2" python scripts/time_driver.py "$1" > /dev/null 2>&1
