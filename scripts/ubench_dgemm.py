"""cuBLAS DGEMM throughput (torch float64 matmul) at the interpolation / Procrustes shapes."""
import torch
torch.backends.cuda.matmul.allow_tf32 = False
for (m, k, n, reps) in [(2048, 256, 2048, 50), (256, 256, 2048, 200), (512, 128, 512, 200), (4096, 4096, 4096, 5),
                        (196608, 300, 300, 5), (300, 196608, 300, 5)]:
    a = torch.randn(m, k, dtype=torch.float64, device="cuda")
    b = torch.randn(k, n, dtype=torch.float64, device="cuda")
    for _ in range(3):
        c = a @ b
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        c = a @ b
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"{m}x{k} @ {k}x{n}: {ms*1e3:.1f} us  {2*m*n*k/ms/1e9:.2f} TFLOP/s")
