"""Batched 256^3 complex GEMM: this library's DMMA kernel (each algo) vs cuBLAS (torch.bmm)."""
import sys; sys.path.insert(0, '/root/repo')
import torch
from paper_2508_19138_b200 import _lib
dev = torch.device('cuda')
b, n = (int(x) for x in (sys.argv[1:3] if len(sys.argv) > 2 else (128, 256)))
g = torch.Generator(device=dev).manual_seed(0)
r = lambda: torch.complex(torch.randn(b, n, n, generator=g, device=dev, dtype=torch.float64),
                          torch.randn(b, n, n, generator=g, device=dev, dtype=torch.float64))
A, B = r(), r()
D = torch.empty_like(A)
lib = _lib.load()
fl = 8.0 * n ** 3 * b
def timeit(fn, reps=10):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
ms = timeit(lambda: torch.bmm(A, B, out=D))
print(f"cuBLAS bmm {b}x{n}^3: {ms:.3f} ms {fl / ms / 1e9:.2f} TFLOP/s", flush=True)
for algo in [int(a) for a in (sys.argv[3].split(",") if len(sys.argv) > 3 else ["2", "3", "0"])]:
    assert lib.negf_set_gemm_algo(algo) == 0, algo
    ms = timeit(lambda: lib.negf_zgemm_batched(n, n, n, b, 1.0, 0.0, A.data_ptr(), n * n, n, 0, B.data_ptr(), n * n, n, 0,
                                               0.0, 0.0, None, 0, n, D.data_ptr(), n * n, n, _lib.stream_ptr()))
    print(f"negf algo {algo}: {ms:.3f} ms {fl / ms / 1e9:.2f} TFLOP/s (algorithmic)", flush=True)
lib.negf_set_gemm_algo(2)
