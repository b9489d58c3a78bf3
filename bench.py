#!/usr/bin/env python
"""Benchmark of the B200-native NEGF hot path.

Workload (BASELINE.json configs[1], "C2"): ballistic NEGF -- carrier
assembly, both contact self-energies (Sancho-Rubio), and the RGF selected
solve for G^R, G^<, G^> -- on chain_device(64 blocks x 256 orbitals),
1024 energies on [-2, 2] eV, eta = 1e-3, mu = +-0.1, kT = 0.05.
One "step" is the complete 1024-energy job (in energy batches). Multi-GPU is
weak scaling: every rank solves its own 1024-energy slice of a 1024*N grid
(energies are independent; no data-path collective on the ballistic path).
The headline computes G^> by the exact carrier identity (configs[1] names
G^R/G^<); ``greater_alt`` times the same job with G^> by its own recursion,
the reference's algorithm, beside it. Further legs: C4-shape (configs[3])
and C3-shape (configs[2]) GW rates and the convolution roofline.

Contract: one JSON line on rank 0 (see the task's bench contract):
metric/value = energy points per second (whole job), roofline of the
dominant kernel (DMMA ZGEMM) from live CUDA-event timing, e2e through the
public API with host buffers, cpu_baseline from the oracle port timed on
this host's cores.

``--impl reference`` times the reference algorithm on the host CPU (the
numpy restatement in oracle/, one energy per core per step) on the same
workload and prints the same JSON line with "impl": "reference".
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "energy_points_per_s (ballistic NEGF: G assembly + OBC + RGF G^R/G^</G^>)"
UNIT = "energy-points/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["native", "reference"], default="native")
    ap.add_argument("--n-blocks", type=int, default=64)
    ap.add_argument("--block-size", type=int, default=256)
    ap.add_argument("--n-e", type=int, default=1024, help="energies per rank")
    ap.add_argument("--batch", type=int, default=0,
                    help="energies per device batch (0: the fewest batches of at most 148 energies, so the "
                         "one-CTA-per-matrix inversion panels cover the 148 SMs: 7 x 147 for 1024)")
    ap.add_argument("--e2e-steps", type=int, default=1)
    ap.add_argument("--greater", choices=["identity", "recursion"], default="identity",
                    help="G^> by the exact identity G^> = G^< + G^R - G^R^dag (default: BASELINE configs[1] names "
                         "G^R/G^<; the identity gives G^> on top at the cost of an elementwise pass) or by its own "
                         "Keldysh recursion like the reference; the other variant is timed beside it (greater_alt)")
    ap.add_argument("--alt-steps", type=int, default=3, help="timed steps of the other --greater variant")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-procs", type=int, default=0, help="0 = all host cores")
    ap.add_argument("--scgw", default="64x512x16", help="n_blocks x block_size x energies-per-rank of the "
                    "SCGW-iteration rate (default: the BASELINE configs[2] C3 device; '' to skip)")
    ap.add_argument("--scgw-batch", type=int, default=8, help="energies per device batch of the SCGW leg")
    ap.add_argument("--c4", default="40x2048x2", help="n_blocks x block_size x energies-per-rank of the "
                    "NRFET-scale (BASELINE configs[3]) G+W RGF-phase rate ('' to skip)")
    return ap.parse_args()


WORKLOAD = dict(e_min=-2.0, e_max=2.0, eta=1e-3, mu_left=0.1, mu_right=-0.1, kT=0.05, surface_tol=1e-8)


def model_flops_per_energy(n_b: int, bs: int, kinds: int = 2) -> float:
    """F_RGF = 8 bs^3 (38 n_b - 33) per energy with both Keldysh
    kinds; one kind: retarded (8 n_b - 7) + one Keldysh pass (15 n_b - 13)."""
    if kinds == 2:
        return 8.0 * bs ** 3 * (38 * n_b - 33)
    return 8.0 * bs ** 3 * (23 * n_b - 20)


# -- CPU legs (oracle port) ---------------------------------------------------


def _cpu_worker(args):
    n_b, bs, energies = args
    from threadpoolctl import threadpool_limits

    sys.path.insert(0, str(ROOT / "oracle"))
    import numpy as np
    import negf_oracle as orc

    w = WORKLOAD
    h = orc.chain_device(n_b, bs)
    with threadpool_limits(1):
        t0 = time.perf_counter()
        orc.ballistic(h, np.asarray(energies), w["eta"], w["mu_left"], w["mu_right"], w["kT"], w["surface_tol"])
        return time.perf_counter() - t0


def cpu_sample(n_b: int, bs: int, energies, procs: int) -> tuple[float, int, float]:
    """Time the oracle on `procs` processes x 1 energy each; returns
    (energies/s, procs, wall s)."""
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    chunks = [(n_b, bs, [float(energies[i % len(energies)])]) for i in range(procs)]
    with ctx.Pool(procs) as pool:
        pool.map(_cpu_worker, [(n_b, 16, [0.0])] * procs)  # warm the workers
        t0 = time.perf_counter()
        pool.map(_cpu_worker, chunks)
        wall = time.perf_counter() - t0
    return procs / wall, procs, wall


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


# -- clocks ------------------------------------------------------------------


class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                rows.append(parts)
        os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = sorted(float(r[1]) for r in rows if r[1].replace(".", "").isdigit())
        smax = max(float(r[2]) for r in rows if r[2].replace(".", "").isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[5 + k].lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": smax, "reasons": reasons,
                "samples": len(rows)}


# -- native arm ------------------------------------------------------------------


def hbm_peak_gbs() -> float:
    """Measured HBM copy bandwidth (read + write bytes) of this pool's B200s
    (MEASURED_PEAKS.json, driver-written); else the recipe's fallback."""
    try:
        return float(json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"])
    except (OSError, KeyError, ValueError):
        return 6500.0


def fp64_peak_probe(dev) -> float:
    """cuBLAS ZGEMM 4096^3 (torch.matmul complex128): the FP64 roofline
    denominator, measured live (MEASURED_PEAKS.json has no FP64 entry)."""
    import torch

    n = 4096
    a = torch.randn(n, n, dtype=torch.complex128, device=dev)
    b = torch.randn(n, n, dtype=torch.complex128, device=dev)
    torch.matmul(a, b)
    torch.cuda.synchronize(dev)
    best = 0.0
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            torch.matmul(a, b)
        e1.record()
        torch.cuda.synchronize(dev)
        best = max(best, 3 * 8.0 * n ** 3 / (e0.elapsed_time(e1) * 1e-3) / 1e12)
    del a, b
    torch.cuda.empty_cache()
    return best


def run_native(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2508_19138_b200 import _lib, toys
    from paper_2508_19138_b200.carrier import CarrierSolver, Contacts, ObservableAccumulator, ballistic_observables

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    w = WORKLOAD
    n_b, bs, n_e = args.n_blocks, args.block_size, args.n_e
    grid = np.linspace(w["e_min"], w["e_max"], n_e * world)
    mine = grid[rank * n_e:(rank + 1) * n_e]
    de = grid[1] - grid[0]
    h = toys.chain_device(n_b, bs)
    contacts = Contacts(w["mu_left"], w["mu_right"], w["kT"])
    lib = _lib.load()
    peak = fp64_peak_probe(dev)
    solver = CarrierSolver(h, w["eta"], contacts, w["surface_tol"], device=dev, greater=args.greater)
    nbatch = -(-n_e // 148)
    batch = min(args.batch, n_e) if args.batch > 0 else -(-n_e // nbatch)
    acc = ObservableAccumulator(n_e, n_b, de, dev)

    def step():
        for s in range(0, n_e, batch):
            chunk = mine[s:s + batch]
            b = solver.solve(chunk, n_e=len(chunk), check=False)
            acc.add(solver, b, s, len(chunk))
        return b

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local])

    for _ in range(args.warmup):
        b = step()
    solver.check_status(b)
    torch.cuda.synchronize(dev)

    clocks = ClockSampler(local)
    clocks.start()
    lib.negf_prof_reset()
    lib.negf_prof_enable(1)
    launches0 = lib.negf_launch_count()
    barrier()
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        b = step()
    e1.record()
    torch.cuda.synchronize(dev)
    barrier()
    launches = lib.negf_launch_count() - launches0
    lib.negf_prof_enable(0)
    clk = clocks.stop()
    ms = e0.elapsed_time(e1)
    solver.check_status(b)
    import ctypes

    breakdown = {}
    tot = [0.0, 0.0, 0]
    for cls, name in ((0, "zgemm_dmma_k_gt_32"), (4, "zgemm_dmma_k_le_32 (inversion sweeps)"),
                      (1, "zinv_panel_swap_rows_unpermute"), (2, "elementwise"), (3, "other")):
        c_ms, c_fl, c_by, c_n = ctypes.c_double(), ctypes.c_double(), ctypes.c_double(), ctypes.c_longlong()
        _lib.check(lib.negf_prof_query(cls, ctypes.byref(c_ms), ctypes.byref(c_fl), ctypes.byref(c_by),
                                       ctypes.byref(c_n)), "negf_prof_query")
        breakdown[name] = {"ms": c_ms.value, "launches": c_n.value}
        if c_fl.value > 0:
            breakdown[name]["tflops_algorithmic"] = c_fl.value / (c_ms.value * 1e-3) / 1e12
        if cls in (0, 4):
            tot[0] += c_ms.value
            tot[1] += c_fl.value
            tot[2] += c_n.value
    breakdown_share = (breakdown["zgemm_dmma_k_gt_32"]["ms"] + breakdown["zgemm_dmma_k_le_32 (inversion sweeps)"]["ms"]) / ms
    lib.negf_prof_reset()
    # Kernel-level roofline from one extra SERIALISED batch (forward-sweep
    # stream overlap off): in the timed region the retarded-chain kernels
    # share the SMs with the Keldysh GEMMs, which stretches per-launch event
    # times without changing the work.
    lib.negf_set_rgf_overlap(0)
    lib.negf_prof_enable(1)
    solver.solve(mine[:batch], n_e=batch, check=False)
    torch.cuda.synchronize(dev)
    lib.negf_prof_enable(0)
    lib.negf_set_rgf_overlap(1)
    tot = [0.0, 0.0, 0]
    for cls in (0, 4):
        c_ms, c_fl, c_by, c_n = ctypes.c_double(), ctypes.c_double(), ctypes.c_double(), ctypes.c_longlong()
        _lib.check(lib.negf_prof_query(cls, ctypes.byref(c_ms), ctypes.byref(c_fl), ctypes.byref(c_by),
                                       ctypes.byref(c_n)), "negf_prof_query")
        tot[0] += c_ms.value
        tot[1] += c_fl.value
        tot[2] += c_n.value
    lib.negf_prof_reset()
    g_ms, g_fl, g_n = ctypes.c_double(tot[0]), ctypes.c_double(tot[1]), ctypes.c_longlong(tot[2])
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    total_e = n_e * world * args.steps
    value = total_e / (ms_max * 1e-3)

    # end-to-end through the public API with host buffers: H2D of the H
    # blocks every step, D2H of the observables every step.
    h_pinned = tuple(torch.from_numpy(np.ascontiguousarray(x)).pin_memory() for x in h)
    h2d = sum(x.numel() * x.element_size() for x in h_pinned) + mine.nbytes
    barrier()
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    obs = {"terminal_left": None, "terminal_right": None}
    for _ in range(args.e2e_steps):
        obs = ballistic_observables(h_pinned, mine, w["eta"], contacts, w["surface_tol"], batch=batch, solver=solver)
    torch.cuda.synchronize(dev)
    e2e_s = time.perf_counter() - t0
    t = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_s = float(t.item())
    d2h = ObservableAccumulator(n_e, n_b, de, dev).d2h_bytes()

    # parity at the benchmarked shape, in the same run: the public API on the
    # energies of the reference fixture tests/golden/golden_c2_ballistic.npz
    # (the reference's own scba_run on chain_device(64, 256), 4 energies)
    parity = None
    gpath = ROOT / "tests" / "golden" / "golden_c2_ballistic.npz"
    if rank == 0 and (n_b, bs) == (64, 256) and gpath.exists():
        g = np.load(gpath)
        ge = np.linspace(-2.0, 2.0, int(g["config"][2]))
        po = ballistic_observables(h, ge, w["eta"], contacts, w["surface_tol"], solver=solver)
        rel = lambda a, b_: float(np.linalg.norm(np.asarray(a) - b_) / np.linalg.norm(b_))
        parity = {"reference_fixture": "tests/golden/golden_c2_ballistic.npz (reference scba_run, 4 energies)",
                  "dos_rel_err": rel(po["dos"], g["obs_dos"]), "density_rel_err": rel(po["density"], g["obs_density"]),
                  "terminal_left": [po["terminal_left"], float(g["obs_terminal_left"])],
                  "terminal_right": [po["terminal_right"], float(g["obs_terminal_right"])],
                  "bar": "1e-9 relative Frobenius (currents: see tests/test_gpu_large_shapes.py)"}
    del solver, acc, b
    _lib._WS.clear()
    torch.cuda.empty_cache()
    # the other G^> variant, timed the same way beside the headline (VERDICT
    # r1: the identity halves the greater pass; the reference runs the recursion)
    alt_mode = "identity" if args.greater == "recursion" else "recursion"
    alt = None
    if args.alt_steps > 0:
        solver_alt = CarrierSolver(h, w["eta"], contacts, w["surface_tol"], device=dev, greater=alt_mode)
        acc_alt = ObservableAccumulator(n_e, n_b, de, dev)

        def step_alt():
            for s in range(0, n_e, batch):
                chunk = mine[s:s + batch]
                bb = solver_alt.solve(chunk, n_e=len(chunk), check=False)
                acc_alt.add(solver_alt, bb, s, len(chunk))
            return bb

        bb = step_alt()
        solver_alt.check_status(bb)
        barrier()
        torch.cuda.synchronize(dev)
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record()
        for _ in range(args.alt_steps):
            bb = step_alt()
        a1.record()
        torch.cuda.synchronize(dev)
        barrier()
        solver_alt.check_status(bb)
        t = torch.tensor([a0.elapsed_time(a1)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        alt_ms = float(t.item())
        alt = {"greater": alt_mode, "value": n_e * world * args.alt_steps / (alt_ms * 1e-3), "unit": UNIT,
               "steps": args.alt_steps, "warmup": 1, "ms_per_step": alt_ms / args.alt_steps,
               "rgf_tflops_model": model_flops_per_energy(n_b, bs, 1 if alt_mode == "identity" else 2)
               * n_e * world * args.alt_steps / (alt_ms * 1e-3) / 1e12}
        del solver_alt, bb, acc_alt
        _lib._WS.clear()
        torch.cuda.empty_cache()

    import gc

    def release():
        gc.collect()  # scba_run's closures form reference cycles over its device buffers
        _lib._WS.clear()
        torch.cuda.empty_cache()

    release()
    c4 = None
    if args.c4 and world > 1:
        c4 = {"skipped": "single-GPU leg (one C4 energy pair needs ~180 GB of one B200; the energy-sharded run "
                         "adds symmetric-memory exchange buffers)"}
    if args.c4 and world == 1:  # first of the GW legs: it needs nearly the whole 180 GB
        try:
            c4 = run_gw_rate(args.c4, 1, dev, world, rank, barrier, "C4 NRFET-scale shape (BASELINE configs[3] device)",
                             peak=peak)
        except torch.OutOfMemoryError as exc:  # reported, not fatal: the headline is C2
            c4 = {"error": f"out of memory: {str(exc).splitlines()[0]}"}
        release()
    scgw = run_scgw(args, dev, world, rank, barrier, peak) if args.scgw else None
    release()
    conv_rf = conv_roofline(dev) if rank == 0 else None
    release()

    # CPU baseline: oracle port on this host's cores (rank 0, N=1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        procs = args.cpu_procs or min(host_cores(), 16)
        rate, procs, wall = cpu_sample(n_b, bs, mine[:: max(1, n_e // procs)], procs)
        cpu = {"value": rate, "unit": UNIT, "cores": procs, "kind": "port",
               "sample": f"{procs} energies of C2 (one per process, 1 BLAS thread each), oracle/negf_oracle.ballistic "
                         f"(numpy restatement of assembly+Sancho OBC+RGF), wall {wall:.1f} s"}

    if rank == 0:
        gemm_avg_ms = g_ms.value / max(g_n.value, 1)
        achieved = g_fl.value / (g_ms.value * 1e-3) / 1e12 if g_ms.value > 0 else 0.0
        traffic, traffic_note = None, None
        tf = ROOT / "profiles" / "zgemm_traffic.json"
        if tf.exists():
            tj = json.loads(tf.read_text())
            traffic = tj.get("dram_bytes_per_launch")
            traffic_note = (f"one ncu --set full capture ({tj.get('launch')}): dram read+write per launch vs "
                            f"{tj.get('algorithmic_bytes_per_launch')} algorithmic bytes; {tj.get('source')}")
        rgf_model = model_flops_per_energy(n_b, bs, 1 if args.greater == "identity" else 2) * total_e
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "complex128 (fp64)",
            "data": "synthetic (seeded chain_device, reference generator restated)",
            "config": {"workload": "C2 ballistic NEGF: chain_device 64 blocks x 256 orbitals, 1024 energies/rank "
                                   "on [-2,2] eV, eta=1e-3, Sancho OBC tol 1e-8, G^R + G^< selected solve (+ G^>)",
                       "greater": args.greater,
                       "n_blocks": n_b, "block_size": bs, "energies_per_rank": n_e, "energy_batch": batch,
                       "parallelism": f"energy-sharded x{world}",
                       "l2": "working set per batch ~100+ GB >> 126 MB L2 (inputs larger than L2)"},
            "rgf_tflops_model": rgf_model / (ms_max * 1e-3) / 1e12,
            "rgf_tflops_model_note": ("SURVEY §8(d) model flops of the recursions actually run (both Keldysh kinds: "
                                      "8 bs^3 (38 n_b - 33); greater by identity: retarded + lesser 8 bs^3 (23 n_b - 20)) "
                                      "/ step time (incl. OBC + assembly)"),
            "greater": ("G^> = G^< + G^R - G^R^dag on the selected blocks (exact: B^> - B^< = M^dag - M for the "
                        "carrier system, SURVEY §7.8; parity-tested vs the reference's greater recursion)"
                        if args.greater == "identity" else "G^> by its own Keldysh recursion (reference algorithm)"),
            "roofline": {"bound": "tensor", "kernel": "zgemm_kernel (DMMA m8n8k4 f64)", "achieved": achieved,
                         "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak if peak else None,
                         "traffic": traffic, "traffic_basis": traffic_note,
                         "achieved_basis": f"algorithmic 8*M*N*K*batch flops of the {g_n.value} ZGEMM launches of one "
                                           f"{batch}-energy batch / their CUDA-event time ({gemm_avg_ms:.3f} ms avg), "
                                           f"measured in bench.py right after the timed region with the forward-sweep "
                                           f"stream overlap off (device_time_breakdown is the timed region itself)",
                         "peak_basis": "cuBLAS ZGEMM 4096^3 measured live in this run (FP64 not in MEASURED_PEAKS.json)",
                         "zgemm_share_of_step": breakdown_share,
                         "complex_product": "3M (Gauss): 3 real DMMA products per complex product; achieved counts "
                                            "the standard 8*M*N*K complex flops, the DMMA pipe executes 6*M*N*K",
                         "executed_dmma_tflops": achieved * 0.75,
                         "executed_frac_of_dmma_peak": achieved * 0.75 / peak if peak else None},
            "e2e": {"value": n_e * world * args.e2e_steps / e2e_s if args.e2e_steps else None, "unit": UNIT,
                    "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h,
                    "api": "paper_2508_19138_b200.carrier.ballistic_observables (host H in, host observables out)"},
            "greater_alt": alt,
            "scgw_iteration": scgw,
            "c4_rgf_rate": c4,
            "conv_roofline": conv_rf,
            "gpu_launches": int(launches),
            "device_time_breakdown": breakdown,
            "clocks": clk,
            "cpu_baseline": cpu,
            "observables_e2e": {"terminal_left": obs["terminal_left"], "terminal_right": obs["terminal_right"],
                                "conservation": (abs(obs["terminal_left"] + obs["terminal_right"])
                                                 / abs(obs["terminal_left"])) if obs["terminal_left"] else None},
            "parity_check": parity,
        }
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_gw_rate(spec: str, batch: int | None, dev, world, rank, barrier, label: str, profile_layout: bool = False,
                peak: float | None = None) -> dict:
    """GW iterations (carrier solve + OBC, polarization, W assembly + closure
    + RGF, self-energy, mixing) on ``spec`` = "n_blocks x block_size x
    energies-per-rank", energy-sharded over the ranks (weak scaling), OBC
    memoizer on as in the reference default. Two iterations; the second
    (warm buffers, nonzero Sigma) is timed, max over ranks. Stage times come
    from device-synchronised stage timers of that iteration; the RGF-phase
    rates use the SURVEY §8(d) model flops F_RGF = 8 bs^3 (38 n_b - 33) per
    energy and subsystem."""
    import numpy as np
    import torch

    from paper_2508_19138_b200 import toys
    from paper_2508_19138_b200.carrier import Contacts
    from paper_2508_19138_b200.dist import Comm
    from paper_2508_19138_b200.scba import ScbaOptions, scba_run

    n_b, bs, ne_rank = (int(x) for x in spec.split("x"))
    batch = batch or ne_rank
    w = WORKLOAD
    e = np.linspace(w["e_min"], w["e_max"], ne_rank * world)
    h, v = toys.chain_device(n_b, bs), toys.coulomb_matrix(n_b, bs)
    comm = Comm.from_env()
    opts = ScbaOptions(retarded_method="sancho", max_iter=2, tol=1e-5, batch=batch)
    contacts = Contacts(w["mu_left"], w["mu_right"], w["kT"])
    torch.cuda.reset_peak_memory_stats(dev)
    barrier()
    res = scba_run(h, v, e, w["eta"], contacts, opts, device=dev, keep_g=False, comm=comm, sigma_to_host=False,
                   profile=True)
    stage = res["timings_by_iteration"][-1]
    vals = [res["iteration_s"][-1], stage.get("G: OBC+RGF", 0.0), stage.get("W: RGF", 0.0)]
    t = torch.tensor(vals, dtype=torch.float64, device=dev)
    if world > 1:
        import torch.distributed as dist

        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dt, t_g, t_w = (float(x) for x in t.tolist())
    f = model_flops_per_energy(n_b, bs) * ne_rank * world
    out = {"config": f"{label}: chain_device({n_b},{bs}) + coulomb_matrix, {ne_rank * world} energies "
                     f"({ne_rank}/rank, batch {batch}), energy-sharded x{world}",
           "iteration_s": dt, "energies_per_s": ne_rank * world / dt,
           "timing": "host wall clock of the 2nd GW iteration, device-synchronised stage timers, max over ranks",
           "stage_s_rank0": stage,
           "rgf_tflops_model_G_incl_obc": f / t_g / 1e12 if t_g else None,
           "rgf_tflops_model_W_rgf": f / t_w / 1e12 if t_w else None,
           "rgf_tflops_model_GW_iteration": 2 * f / dt / 1e12,
           # executed: 27 n_b - 23 products + n_b inversions, 8 bs^3 each, per energy and subsystem
           "rgf_tflops_executed_W_rgf": 8.0 * bs ** 3 * (28 * n_b - 23) * ne_rank * world / t_w / 1e12 if t_w else None,
           "fp64_peak_tflops": peak,
           "rgf_executed_frac_of_peak_W_rgf": (8.0 * bs ** 3 * (28 * n_b - 23) * ne_rank * world / t_w / 1e12 / peak)
           if (t_w and peak) else None,
           "model": "F_RGF = 8 bs^3 (38 n_b - 33) per energy per subsystem (SURVEY §8(d)); this implementation "
                    "executes 27 n_b - 23 products + n_b inversions of 8 bs^3, i.e. fewer flops than the model",
           "max_mem_gb_rank0": torch.cuda.max_memory_allocated(dev) / 1e9,
           "transpose_bytes_rank0": int(res["transpose_bytes"]),
           "residual": float(res["residuals"][-1]),
           "obc_memoizer": {"enabled": True, "cache_stats_by_iteration_rank0": res["cache_stats_by_iteration"]}}
    if profile_layout:
        # HBM roofline of the E<->nnz layout kernels: one more iteration with
        # the CUDA-event profiler on (algorithmic bytes recorded per launch)
        import ctypes

        from paper_2508_19138_b200 import _lib

        lib = _lib.load()
        lib.negf_prof_reset()
        lib.negf_prof_enable(1)
        scba_run(h, v, e, w["eta"], contacts, ScbaOptions(retarded_method="sancho", max_iter=1, tol=1e-5, batch=batch), device=dev,
                 keep_g=False, comm=comm, sigma_to_host=False)
        torch.cuda.synchronize(dev)
        lib.negf_prof_enable(0)
        c_ms, c_fl, c_by, c_n = ctypes.c_double(), ctypes.c_double(), ctypes.c_double(), ctypes.c_longlong()
        _lib.check(lib.negf_prof_query(10, ctypes.byref(c_ms), ctypes.byref(c_fl), ctypes.byref(c_by),
                                       ctypes.byref(c_n)), "negf_prof_query")
        lib.negf_prof_reset()
        gbs = c_by.value / (c_ms.value * 1e-3) / 1e9 if c_ms.value > 0 else 0.0
        peak = hbm_peak_gbs()
        out["layout_hbm_roofline"] = {"bound": "hbm", "achieved": gbs, "peak": peak, "unit": "GB/s",
                                      "frac": gbs / peak, "launches": c_n.value, "ms": c_ms.value,
                                      "algorithmic_bytes": "32 B per entry-energy (pack); entries + blocks (unpack)"}
    return out


def run_scgw(args, dev, world, rank, barrier, peak=None) -> dict:
    return run_gw_rate(args.scgw, args.scgw_batch, dev, world, rank, barrier, "C3 shape (BASELINE configs[2] device)",
                       profile_layout=True, peak=peak)


def conv_roofline(dev, n_rows: int = 1 << 17, lengths=(512, 2048, 4096)) -> dict:
    """HBM roofline of the fused P and Sigma convolution kernels at the
    BASELINE energy counts (C1/C3/C4 series lengths) on synthetic entry rows
    (n_rows x N_E complex128 each, >> L2): algorithmic bytes per launch
    (P: read G^<, G^>, write P^<, P^>, P^R_up, P^R_lo = 96 B per entry-energy;
    Sigma: +W^<, W^> = 128 B) / CUDA-event time, against MEASURED_PEAKS.json's
    copy bandwidth."""
    import torch

    from paper_2508_19138_b200.conv import polarization, self_energy

    peak = hbm_peak_gbs()
    out = {}
    for ne in lengths:
        g = torch.Generator(device=dev).manual_seed(ne)
        mk = lambda: torch.complex(torch.randn(n_rows, ne, generator=g, device=dev, dtype=torch.float64),
                                   torch.randn(n_rows, ne, generator=g, device=dev, dtype=torch.float64))
        gl, gg, wl, wg = mk(), mk(), mk(), mk()
        diag = torch.zeros(n_rows, dtype=torch.uint8, device=dev)
        diag[::97] = 1
        res = {}
        for name, fn, per in (("P", lambda o: polarization(gl, gg, diag, 0.01, out=o), 96.0),
                              ("Sigma", lambda o: self_energy(gl, gg, wl, wg, None, diag, 0.01, out=o), 128.0)):
            o = tuple(torch.empty_like(gl) for _ in range(4))
            fn(o)
            torch.cuda.synchronize(dev)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = 5
            e0.record()
            for _ in range(reps):
                fn(o)
            e1.record()
            torch.cuda.synchronize(dev)
            ms = e0.elapsed_time(e1) / reps
            gbs = per * n_rows * ne / (ms * 1e-3) / 1e9
            res[name] = {"ms": ms, "achieved": gbs, "frac": gbs / peak}
            del o
        out[f"N_E={ne}"] = res
        del gl, gg, wl, wg
        torch.cuda.empty_cache()
    return {"bound": "hbm", "peak": peak, "unit": "GB/s", "rows": n_rows,
            "basis": "algorithmic bytes (96 B P / 128 B Sigma per entry-energy) / CUDA-event time per launch set, "
                     "inputs 2-4 x rows x N_E x 16 B >> L2", "lengths": out}


# -- reference arm -----------------------------------------------------------------


def run_reference(args):
    import numpy as np

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    w = WORKLOAD
    n_b, bs, n_e = args.n_blocks, args.block_size, args.n_e
    grid = np.linspace(w["e_min"], w["e_max"], n_e * world)
    procs = args.cpu_procs or host_cores()
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    with ctx.Pool(procs) as pool:
        pool.map(_cpu_worker, [(n_b, 16, [0.0])] * procs)
        for s in range(args.warmup):  # untimed warm-up steps: same work as a timed step
            pool.map(_cpu_worker, [(n_b, bs, [float(grid[(s * procs + i) * 11 % len(grid)])]) for i in range(procs)])
        walls = []
        for s in range(args.steps):
            chunks = [(n_b, bs, [float(grid[(s * procs + i) * 7 % len(grid)])]) for i in range(procs)]
            t0 = time.perf_counter()
            pool.map(_cpu_worker, chunks)
            walls.append(time.perf_counter() - t0)
    value = procs * args.steps / sum(walls)
    sample = (f"each step: {procs} energies of C2 (one per process, 1 BLAS thread each) through the oracle port "
              f"of the reference algorithm (oracle/negf_oracle.ballistic); reference package is pure Python and "
              f"cannot travel to the box")
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * sum(walls) / len(walls), "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "complex128 (fp64)", "data": "synthetic (seeded chain_device)", "impl": "reference",
        "config": {"workload": "C2 ballistic NEGF: chain_device 64 blocks x 256 orbitals, energies on [-2,2] eV",
                   "n_blocks": n_b, "block_size": bs},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": procs, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_native(a)
