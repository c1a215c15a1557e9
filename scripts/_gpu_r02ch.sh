# round-2 session-5 call H: paired two-panel QR: A/B test, cfg4 timing (pair on/off), config parity tests
python -m pytest tests/test_gpu_qr.py -x -q -k "two_panel_pair" 2>&1 | tail -15
for P in 0 1; do echo "== PTB_QR2_PAIR=$P"; PTB_QR2_PAIR=$P python scripts/time_driver.py 4:4 2>&1 | tail -1; done
python -m pytest tests/test_gpu_configs.py tests/test_gpu_sharded.py -x -q 2>&1 | tail -4
