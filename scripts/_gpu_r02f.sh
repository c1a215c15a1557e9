mkdir -p gpurun_out
timeout 600 python scripts/diag_qr.py /tmp/fg3.npz
for v in "PTB_QR=tsqr"; do echo "== $v"; env $v timeout 600 python scripts/diag_qr.py /tmp/fg3.npz run 2>&1 | tail -3; done
timeout 2400 python -m pytest tests -x -q -m gpu > gpurun_out/r02f_tests.log 2>&1; echo tests_rc=$?
tail -15 gpurun_out/r02f_tests.log
