timeout 600 python scripts/diag_qr.py /tmp/fg3.npz
for v in "PTB_QR=tsqr" "PTB_QR=direct"; do echo "== $v"; env $v timeout 600 python scripts/diag_qr.py /tmp/fg3.npz run 2>&1 | tail -3; done
