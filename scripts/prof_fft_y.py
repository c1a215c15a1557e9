"""Minimal driver for ncu of the Fourier interpolation y pass (config 4's fine combine shape):
interpolate_fields_add over `batch` 2048^2 fields from 256^2 coarse fields.
  python scripts/prof_fft_y.py [batch]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes  # noqa: E402

import torch  # noqa: E402

import paratime_b200 as B  # noqa: E402

batch = int(sys.argv[1]) if len(sys.argv) > 1 else 16
ctx = B.Context(0)
nf, nc = 2048, 256
t = B.Transfer(ctx, B.Grid((nc, nc), (1 / nc, 1 / nc)), B.Grid((nf, nf), (1 / nf, 1 / nf)), B.FOURIER)
d = torch.randn((batch, nc, nc), dtype=torch.float64, device="cuda")
base = torch.randn((batch, nf, nf), dtype=torch.float64, device="cuda")
out = torch.empty_like(base)
for _ in range(3):
    B.api.check(B.lib().ptb_interpolate_add_batch(t.h, ctypes.c_size_t(batch), ctypes.c_void_p(d.data_ptr()),
                                                  ctypes.c_void_p(base.data_ptr()), ctypes.c_void_p(out.data_ptr())))
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
B.api.check(B.lib().ptb_interpolate_add_batch(t.h, ctypes.c_size_t(batch), ctypes.c_void_p(d.data_ptr()),
                                              ctypes.c_void_p(base.data_ptr()), ctypes.c_void_p(out.data_ptr())))
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
print(f"interpolate+add {batch} x {nf}^2: {ms:.3f} ms, {batch * nf * nf * 16 / ms / 1e6:.0f} GB/s (base read + out write)")
