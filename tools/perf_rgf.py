"""Quick RGF throughput probe at the C2 shape (synthetic diagonally shifted blocks)."""
import sys, time; sys.path.insert(0, '/root/repo')
import torch
from paper_2508_19138_b200 import selected_solve_batched, _lib
dev = torch.device('cuda')
nb_, bs = int(sys.argv[1]) if len(sys.argv) > 1 else 64, int(sys.argv[2]) if len(sys.argv) > 2 else 256
for ne in [int(x) for x in (sys.argv[3].split(',') if len(sys.argv) > 3 else ['16', '48'])]:
    g = torch.Generator(device=dev).manual_seed(0)
    def r(*s):
        return torch.complex(torch.randn(*s, generator=g, device=dev, dtype=torch.float64),
                             torch.randn(*s, generator=g, device=dev, dtype=torch.float64)) * (1.0 / bs ** 0.5)
    eye = torch.eye(bs, dtype=torch.complex128, device=dev)
    md = r(ne, nb_, bs, bs) + (4 + 1j) * eye
    mu, ml = r(ne, nb_ - 1, bs, bs), r(ne, nb_ - 1, bs, bs)
    bl = (r(ne, nb_, bs, bs), r(ne, nb_ - 1, bs, bs))
    bg = (r(ne, nb_, bs, bs), r(ne, nb_ - 1, bs, bs))
    out = selected_solve_batched(md, mu, ml, bl, bg, symmetrize=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 2
    e0.record()
    for _ in range(reps):
        selected_solve_batched(md, mu, ml, bl, bg, symmetrize=True, out=out, check=False)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    f_exec = 8.0 * bs ** 3 * (28 * nb_ - 23) * ne
    f_model = 8.0 * bs ** 3 * (38 * nb_ - 33) * ne
    print(f"n_b={nb_} bs={bs} n_e={ne}: {ms:.1f} ms/solve  {ne / ms * 1e3:.1f} energies/s  "
          f"exec {f_exec / ms / 1e9:.2f} TFLOP/s  model {f_model / ms / 1e9:.2f} TFLOP/s", flush=True)
    del md, mu, ml, bl, bg, out
    torch.cuda.empty_cache()
