timeout 120 python scripts/diag_world.py 3; echo rc=$?
PTB_PDL=0 timeout 120 python scripts/diag_world.py 3; echo rc_nopdl=$?
