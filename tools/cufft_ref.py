"""Dev calibration: cuFFT (torch.fft) time for the C3 shape (not used by the product)."""
import torch
for L in (28, 30):
    n = 1 << L
    x = torch.randn(n, dtype=torch.complex64, device="cuda")
    y = torch.fft.fft(x)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        y = torch.fft.fft(x)
    e1.record()
    torch.cuda.synchronize()
    print(f"cuFFT c64 2^{L}: {e0.elapsed_time(e1) / 5:.3f} ms")
    del x, y
    torch.cuda.empty_cache()
