"""Energy sharding and the energy <-> entry redistribution (the paper's E<->nnz
transposition) over torch.distributed.

Reference: ``energy_chunks`` (scba.py:243-249), ``transpose_distribution``
(scba.py:342-368) and its 12 calls per iteration (scba.py:1028-1141). The
reference moves every slab to every rank (gather + bcast, fully replicated);
here each rank sends each peer exactly the slab that peer owns, in one
``all_to_all_single`` per quantity (NCCL over NVLink on the GPU box, gloo in
the CPU tests):

* to_entry_major: local (n_entries, n_own_e) columns -> (n_own_entries, N_E)
* to_energy_major: local (n_own_entries, N_E) rows -> (n_entries, n_own_e)

Complex tensors travel as their float64 view.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist


def energy_chunks(n: int, size: int) -> list[slice]:
    """scba.py:243-249: contiguous near-even split."""
    base, rem = divmod(n, size)
    bounds = [0]
    for r in range(size):
        bounds.append(bounds[-1] + base + (1 if r < rem else 0))
    return [slice(bounds[r], bounds[r + 1]) for r in range(size)]


@dataclass
class Comm:
    """Rank/size + process group; size 1 makes every transpose an identity."""

    rank: int = 0
    size: int = 1
    group: object = None

    @classmethod
    def from_env(cls, group=None) -> "Comm":
        if dist.is_available() and dist.is_initialized():
            return cls(dist.get_rank(group), dist.get_world_size(group), group)
        return cls()

    def allreduce_max(self, values: list[float], device) -> list[float]:
        if self.size == 1:
            return list(values)
        t = torch.tensor(values, dtype=torch.float64, device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
        return t.tolist()


class Transposer:
    """E <-> nnz redistribution for one (n_entries, N_E) pattern."""

    def __init__(self, comm: Comm, n_entries: int, n_e: int) -> None:
        self.comm = comm
        self.n_entries, self.n_e = n_entries, n_e
        self.e_sl = energy_chunks(n_e, comm.size)
        self.r_sl = energy_chunks(n_entries, comm.size)
        self.own_e = self.e_sl[comm.rank]
        self.own_r = self.r_sl[comm.rank]
        self.n_own_e = self.own_e.stop - self.own_e.start
        self.n_own_r = self.own_r.stop - self.own_r.start
        self.bytes_moved = 0

    def _a2a(self, send: torch.Tensor, in_splits: list[int], out_splits: list[int]) -> torch.Tensor:
        sr = torch.view_as_real(send).reshape(-1)
        recv = torch.empty(2 * sum(out_splits), dtype=torch.float64, device=send.device)
        dist.all_to_all_single(recv, sr, [2 * s for s in out_splits], [2 * s for s in in_splits],
                               group=self.comm.group)
        self.bytes_moved += 16 * (sum(in_splits) - in_splits[self.comm.rank])
        return torch.view_as_complex(recv.view(-1, 2))

    def to_entry_major(self, cols: torch.Tensor) -> torch.Tensor:
        """(n_entries, n_own_e) -> (n_own_entries, N_E)."""
        if self.comm.size == 1:
            return cols
        P = self.comm.size
        send = cols.contiguous()  # entry-chunk row blocks are contiguous
        in_splits = [(s.stop - s.start) * self.n_own_e for s in self.r_sl]
        out_splits = [self.n_own_r * (s.stop - s.start) for s in self.e_sl]
        recv = self._a2a(send, in_splits, out_splits)
        parts, off = [], 0
        for s in range(P):
            ne_s = self.e_sl[s].stop - self.e_sl[s].start
            parts.append(recv[off:off + self.n_own_r * ne_s].view(self.n_own_r, ne_s))
            off += self.n_own_r * ne_s
        return torch.cat(parts, dim=1)

    def rows_to_full(self, rows: torch.Tensor) -> torch.Tensor:
        """(n_own_entries, N_E) -> (n_entries, N_E) on every rank: the
        replicated result of the reference's to-energy-major transpose
        (scba.py:342-368), needed only by the spatial mode of scba_run where
        every rank solves every energy. One padded all-gather."""
        if self.comm.size == 1:
            return rows
        m = max(s.stop - s.start for s in self.r_sl)
        pad = torch.zeros((m, self.n_e), dtype=rows.dtype, device=rows.device)
        pad[:self.n_own_r] = rows
        bufs = [torch.empty_like(pad) for _ in range(self.comm.size)]
        dist.all_gather([torch.view_as_real(x) for x in bufs], torch.view_as_real(pad), group=self.comm.group)
        self.bytes_moved += 16 * self.n_own_r * self.n_e * (self.comm.size - 1)
        return torch.cat([x[:s.stop - s.start] for x, s in zip(bufs, self.r_sl)])

    def to_energy_major(self, rows: torch.Tensor) -> torch.Tensor:
        """(n_own_entries, N_E) -> (n_entries, n_own_e)."""
        if self.comm.size == 1:
            return rows
        send = torch.cat([rows[:, s].contiguous().view(-1) for s in self.e_sl])
        in_splits = [self.n_own_r * (s.stop - s.start) for s in self.e_sl]
        out_splits = [(s.stop - s.start) * self.n_own_e for s in self.r_sl]
        recv = self._a2a(send, in_splits, out_splits)
        return recv.view(self.n_entries, self.n_own_e)


class PeerEntryMajor:
    """Entry-major arrays in symmetric memory (torch.distributed._symmetric_memory:
    one allocation per rank, every peer's buffer mapped over NVLink), so the
    pack kernel writes each entry row straight into its owner's array
    (negf_pack_lg_p2p) -- the E -> nnz transpose fused with the pack, no
    staging columns and no NCCL all-to-all. One buffer per quantity name,
    (max entry chunk, N_E) complex128, reused across iterations."""

    def __init__(self, tr: "Transposer", device) -> None:
        import torch.distributed._symmetric_memory as symm

        self.tr, self.dev, self.symm = tr, torch.device(device), symm
        rows = max(s.stop - s.start for s in tr.r_sl)
        self.shape = (rows, tr.n_e)
        self.row_start = torch.tensor([s.start for s in tr.r_sl] + [tr.r_sl[-1].stop], dtype=torch.int64,
                                      device=self.dev)
        self._bufs: dict[str, tuple] = {}

    @classmethod
    def try_create(cls, tr: "Transposer", device) -> "PeerEntryMajor | None":
        """The peer path when the setup supports it -- an NCCL process group on
        CUDA devices with symmetric memory (NVLink P2P) -- decided jointly by
        all ranks (MIN over the per-rank outcome); None selects the NCCL
        all-to-all Transposer."""
        group = tr.comm.group or dist.group.WORLD
        ok = 1
        pem = None
        try:
            if dist.get_backend(group) != "nccl" or not torch.cuda.is_available():
                ok = 0
            else:
                pem = cls(tr, device)
                pem.buffer("gl")  # first rendezvous: fails here without symmetric-memory support
        except Exception:  # noqa: BLE001 -- any failure selects the all-to-all path
            ok = 0
        if dist.get_backend(group) == "nccl":
            flag = torch.tensor([ok], dtype=torch.int32, device=device)
            dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=tr.comm.group)
            ok = int(flag.item())
        return pem if ok else None

    def buffer(self, name: str):
        """(local (n_own_entries, N_E) view, device array of the peers' base pointers, handle)."""
        if name not in self._bufs:
            t = self.symm.empty(self.shape, dtype=torch.complex128, device=self.dev)
            group = self.tr.comm.group or dist.group.WORLD
            h = self.symm.rendezvous(t, group.group_name)
            ptrs = torch.tensor(list(h.buffer_ptrs), dtype=torch.int64, device=self.dev)
            self._bufs[name] = (t, ptrs, h)
        t, ptrs, h = self._bufs[name]
        return t[:self.tr.n_own_r], ptrs, h

    def barrier(self) -> None:
        """Stream-ordered cross-rank barrier: every peer's writes into our
        buffers are complete (and ours into theirs) before what follows."""
        if self._bufs:
            next(iter(self._bufs.values()))[2].barrier()

    def count(self, n_cols: int) -> None:
        """Bytes this rank wrote to peers for n_cols energy columns."""
        self.tr.bytes_moved += 16 * n_cols * (self.tr.n_entries - self.tr.n_own_r)


TO_ENTRY_MAJOR = "to_entry_major"
TO_ENERGY_MAJOR = "to_energy_major"


def transpose_distribution(comm: Comm, local_part, direction: str, stats=None, lg: bool = True,
                           full_entry_count: int = 0):
    """scba.py:342-368, same signature and semantics: ``to_entry_major``
    gathers every rank's energy columns (n_entries, n_own_e) into the
    replicated (n_entries, N_E) array, ``to_energy_major`` gathers every
    rank's entry rows (n_own_entries, N_E) into it; ``stats`` (a
    TranspositionStats) counts the full logical redistribution like
    _count_bytes (scba.py:385-394). ``local_part`` is a numpy array (returned
    as numpy) or a torch tensor (returned on its device). One padded
    all-gather over the process group (NCCL needs CUDA tensors; gloo CPU).

    The hot path does not replicate: scba_run moves each rank only the slab
    it owns (Transposer / the fused peer-memory layout kernels); this drop-in
    is for callers written against the reference."""
    import numpy as np

    from .results import count_transpose_bytes

    if direction not in (TO_ENTRY_MAJOR, TO_ENERGY_MAJOR):
        raise ValueError(f"unknown transpose direction {direction!r}")
    as_np = isinstance(local_part, np.ndarray)
    x = torch.from_numpy(np.ascontiguousarray(local_part, dtype=complex)) if as_np else local_part.contiguous()
    axis = 1 if direction == TO_ENTRY_MAJOR else 0
    if comm.size == 1:
        full = x
    else:
        group = comm.group
        dev = x.device
        if dist.get_backend(group) == "nccl" and dev.type != "cuda":
            dev = torch.device("cuda", torch.cuda.current_device())
        x = x.to(dev)
        n_loc = torch.tensor([x.shape[axis], x.shape[1 - axis]], dtype=torch.int64, device=dev)
        sizes = [torch.empty_like(n_loc) for _ in range(comm.size)]
        dist.all_gather(sizes, n_loc, group=group)
        counts = [int(t[0]) for t in sizes]
        other = int(sizes[0][1])
        if any(int(t[1]) != other for t in sizes):
            raise ValueError("transpose_distribution: ranks disagree on the non-split dimension")
        m = max(counts)
        shape = (other, m) if axis == 1 else (m, other)
        pad = torch.zeros(shape, dtype=torch.complex128, device=dev)
        if axis == 1:
            pad[:, :x.shape[1]] = x
        else:
            pad[:x.shape[0]] = x
        bufs = [torch.empty_like(pad) for _ in range(comm.size)]
        dist.all_gather([torch.view_as_real(b) for b in bufs], torch.view_as_real(pad), group=group)
        parts = [b[:, :c] if axis == 1 else b[:c] for b, c in zip(bufs, counts)]
        full = torch.cat(parts, dim=axis)
    if stats is not None:
        count_transpose_bytes(stats, lg, full.shape[0], full.shape[1], full_entry_count)
    if as_np:
        return full.cpu().numpy()
    return full.to(local_part.device)


def transpose_owned(comm: Comm, local_part: torch.Tensor, direction: str, n_entries: int, n_e: int):
    """The hot-path form of the transposition: an all-to-all in which each
    rank receives only the slab it owns (entry rows for to_entry_major,
    energy columns for to_energy_major) instead of the replicated array."""
    tr = Transposer(comm, n_entries, n_e)
    if direction == TO_ENTRY_MAJOR:
        return tr.to_entry_major(local_part)
    if direction == TO_ENERGY_MAJOR:
        return tr.to_energy_major(local_part)
    raise ValueError(f"unknown transpose direction {direction!r}")
