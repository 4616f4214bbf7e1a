"""PCIe copy rates on the box: 2-D copies of column blocks (H2D / D2H) by
block width, and concurrent H2D + D2H (full duplex?)."""
import ctypes, time, torch
rt = ctypes.CDLL("/usr/local/cuda/lib64/libcudart.so.12")
n = 16384
hA = torch.empty((n, n), dtype=torch.float32, pin_memory=True)
hC = torch.empty((n, n), dtype=torch.float32, pin_memory=True)
d = torch.empty((n, n), dtype=torch.float32, device="cuda")
d2 = torch.empty((n, n), dtype=torch.float32, device="cuda")
s1 = torch.cuda.Stream(); s2 = torch.cuda.Stream()
H2D, D2H = 1, 2
def cp2d(dst, dpitch, src, spitch, w, h, kind, stream):
    r = rt.cudaMemcpy2DAsync(ctypes.c_void_p(dst), ctypes.c_size_t(dpitch), ctypes.c_void_p(src), ctypes.c_size_t(spitch),
                             ctypes.c_size_t(w), ctypes.c_size_t(h), ctypes.c_int(kind), ctypes.c_void_p(stream.cuda_stream))
    assert r == 0, r
def timeit(fn, reps=3):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps
P = n * 4
for cols in (1024, 2048, 4096, 16384):
    def up():
        for c0 in range(0, n, cols):
            cp2d(d.data_ptr() + 4 * c0, P, hA.data_ptr() + 4 * c0, P, 4 * cols, n, H2D, s1)
    def down():
        for c0 in range(0, n, cols):
            cp2d(hC.data_ptr() + 4 * c0, P, d.data_ptr() + 4 * c0, P, 4 * cols, n, D2H, s1)
    tu, td = timeit(up), timeit(down)
    print(f"2-D col blocks {cols:5d} ({4*cols//1024} KB rows): H2D {4*n*n/tu/1e9:.1f} GB/s  D2H {4*n*n/td/1e9:.1f} GB/s", flush=True)
for rows in (1024, 2048):
    def down():
        for r0 in range(0, n, rows):
            for c0 in range(0, n, rows):
                cp2d(hC.data_ptr() + 4 * (r0 * n + c0), P, d.data_ptr() + 4 * (r0 * n + c0), P, 4 * rows, rows, D2H, s1)
    td = timeit(down)
    print(f"D2H {rows}x{rows} blocks: {4*n*n/td/1e9:.1f} GB/s", flush=True)
def both():
    with torch.cuda.stream(s1):
        d.copy_(hA, non_blocking=True)
    with torch.cuda.stream(s2):
        hC.copy_(d2, non_blocking=True)
def up1():
    with torch.cuda.stream(s1):
        d.copy_(hA, non_blocking=True)
def dn1():
    with torch.cuda.stream(s2):
        hC.copy_(d2, non_blocking=True)
tu, td, tb = timeit(up1), timeit(dn1), timeit(both)
print(f"1 GiB H2D alone {tu*1e3:.1f} ms, D2H alone {td*1e3:.1f} ms, both concurrently {tb*1e3:.1f} ms", flush=True)
