"""Pinned device→host copy bandwidth: one 1-D copy of C3's state volume vs the time-chunk 2-D pattern of the host
pipeline (cudaMemcpy2DAsync: 8192 rows of kc·48 B at a host pitch of (K+1)·48 B) — what bounds C3's e2e."""
import time

import torch
from cuda.bindings import runtime as rt

B, K, D = 8192, 10000, 3
row = 2 * D * 8
h = torch.empty((B, K + 1, 2 * D), dtype=torch.float64).pin_memory()
d = torch.empty((B, K + 1, 2 * D), dtype=torch.float64, device="cuda")
s = torch.cuda.Stream()
for kc in (None, 4000, 2000, 1000, 500):
    torch.cuda.synchronize()
    reps = 3
    t0 = time.perf_counter()
    for _ in range(reps):
        if kc is None:
            rt.cudaMemcpyAsync(h.data_ptr(), d.data_ptr(), h.numel() * 8, rt.cudaMemcpyKind.cudaMemcpyDeviceToHost,
                               s.cuda_stream)
        else:
            for k0 in range(0, K + 1, kc):
                n = min(kc, K + 1 - k0)
                # device staging is chunk-contiguous (pitch n·row), host rows at pitch (K+1)·row
                rt.cudaMemcpy2DAsync(h.data_ptr() + k0 * row, (K + 1) * row, d.data_ptr(), n * row, n * row, B,
                                     rt.cudaMemcpyKind.cudaMemcpyDeviceToHost, s.cuda_stream)
    s.synchronize()
    dt = (time.perf_counter() - t0) / reps
    print(f"{'1-D' if kc is None else f'2-D kc={kc}'}: {h.numel() * 8 / dt / 1e9:.1f} GB/s ({dt * 1e3:.1f} ms for "
          f"{h.numel() * 8 / 1e9:.2f} GB)")
