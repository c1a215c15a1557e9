mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_gemm.py -x -q 2>&1 | tail -5
for v in "" "PTB_PDL=0" "PTB_QR=direct" "PTB_QR=blocked"; do
  echo "== $v"; env $v timeout 600 python scripts/diag_procrustes.py 3 2 2>&1 | grep "k=\|Error" 
done
