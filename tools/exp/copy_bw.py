"""Pinned host <-> HBM copy bandwidth: contiguous and 2-D (8 KB rows of a
wide device panel), the shapes of the e2e path's input upload and output
download."""
import ctypes
import torch

n = 1 << 30
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
def t(fn, reps=3):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); e1.synchronize()
    return e0.elapsed_time(e1) / reps
ms = t(lambda: d.copy_(h, non_blocking=True)); print(f"H2D contiguous 1 GiB: {n / ms / 1e6:.1f} GB/s")
ms = t(lambda: h.copy_(d, non_blocking=True)); print(f"D2H contiguous 1 GiB: {n / ms / 1e6:.1f} GB/s")
# 2-D: 8192 rows x 8192 bytes out of a device panel with ld 65536+16
cudart = ctypes.CDLL("libcudart.so") if False else None
dp = torch.empty(8192 * (65536 + 16), dtype=torch.uint8, device="cuda")
hp = torch.empty(8192 * 8192, dtype=torch.uint8, pin_memory=True)
lib = ctypes.CDLL(torch._C.__file__.replace("_C.cpython-312-x86_64-linux-gnu.so", "lib/libcudart.so.12")) if False else None
import cuda.bindings.runtime as rt
s = torch.cuda.current_stream().cuda_stream
def c2d():
    err, = rt.cudaMemcpy2DAsync(hp.data_ptr(), 8192, dp.data_ptr(), 65536 + 16, 8192, 8192,
                                rt.cudaMemcpyKind.cudaMemcpyDeviceToHost, s)
ms = t(c2d); print(f"D2H 2-D 8192 x 8 KB rows (ld 64 KB): {8192 * 8192 / ms / 1e6:.1f} GB/s")
def c2d_h2d():
    err, = rt.cudaMemcpy2DAsync(dp.data_ptr(), 65536 + 16, hp.data_ptr(), 8192, 8192, 8192,
                                rt.cudaMemcpyKind.cudaMemcpyHostToDevice, s)
ms = t(c2d_h2d); print(f"H2D 2-D 8192 x 8 KB rows: {8192 * 8192 / ms / 1e6:.1f} GB/s")
# both directions at once
s2 = torch.cuda.Stream()
def both():
    d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2 = hp
        err, = rt.cudaMemcpy2DAsync(hp.data_ptr(), 8192, dp.data_ptr(), 65536 + 16, 8192, 8192,
                                    rt.cudaMemcpyKind.cudaMemcpyDeviceToHost, s2.cuda_stream)
    torch.cuda.current_stream().wait_stream(s2)
ms = t(both); print(f"H2D 1 GiB + D2H 64 MiB 2-D concurrently: {ms:.2f} ms")
