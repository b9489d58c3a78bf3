"""Host logic of the energy-sharded path at world size 2 on CPU (gloo):
the E <-> nnz all-to-all transposes against the reference's replicated
gather semantics (scba.py:342-368) and energy_chunks (scba.py:243-249)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2508_19138_b200.dist import Comm, Transposer, energy_chunks


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n_entries, n_e, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = Comm.from_env()
        tr = Transposer(comm, n_entries, n_e)
        rng = np.random.default_rng(0)
        full = rng.standard_normal((n_entries, n_e)) + 1j * rng.standard_normal((n_entries, n_e))
        cols = torch.from_numpy(np.ascontiguousarray(full[:, tr.own_e]))
        rows = tr.to_entry_major(cols)
        ok1 = np.array_equal(rows.numpy(), full[tr.own_r])
        back = tr.to_energy_major(rows)
        ok2 = np.array_equal(back.numpy(), full[:, tr.own_e])
        # spatial mode of scba_run: every rank gets all entry rows (replicated
        # to-energy-major result of the reference, scba.py:342-368)
        ok2 = ok2 and np.array_equal(tr.rows_to_full(rows).numpy(), full)
        red = comm.allreduce_max([float(rank), -float(rank)], torch.device("cpu"))
        # reference-signature drop-in (scba.py:342-368): replicated result +
        # TranspositionStats counts, numpy in -> numpy out
        from paper_2508_19138_b200.dist import TO_ENERGY_MAJOR, TO_ENTRY_MAJOR, transpose_distribution
        from paper_2508_19138_b200.results import TranspositionStats

        st = TranspositionStats()
        r1 = transpose_distribution(comm, full[:, tr.own_e], TO_ENTRY_MAJOR, st, True, 2 * n_entries)
        r2 = transpose_distribution(comm, full[tr.own_r], TO_ENERGY_MAJOR, st, False)
        ok2 = ok2 and isinstance(r1, np.ndarray) and np.array_equal(r1, full) and np.array_equal(r2, full)
        ok2 = ok2 and st.lg_bytes == 16 * n_entries * n_e and st.lg_full_bytes == 32 * n_entries * n_e
        ok2 = ok2 and st.other_bytes == 16 * n_entries * n_e and st.lg_ratio() == 0.5
        q.put((rank, ok1, ok2, red, tr.bytes_moved))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n_entries,n_e", [(2, 37, 11), (2, 8, 2), (2, 101, 64), (3, 37, 11), (4, 101, 64),
                                                 (4, 23808 // 16, 128)])
def test_alltoall_transposes(world, n_entries, n_e):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n_entries, n_e, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok1, ok2, red, moved in res:
        assert ok1 and ok2, rank
        assert red == [float(world - 1), 0.0]
        assert moved > 0


def test_energy_chunks_match_reference_rule():
    # scba.py:243-249: near-even contiguous split, remainder to the first ranks
    assert energy_chunks(10, 3) == [slice(0, 4), slice(4, 7), slice(7, 10)]
    assert energy_chunks(2, 4) == [slice(0, 1), slice(1, 2), slice(2, 2), slice(2, 2)]
    assert sum(s.stop - s.start for s in energy_chunks(1023, 8)) == 1023


def test_serial_comm_transposes_are_identity():
    tr = Transposer(Comm(), 9, 5)
    x = torch.zeros(9, 5, dtype=torch.complex128)
    assert tr.to_entry_major(x) is x and tr.to_energy_major(x) is x and tr.rows_to_full(x) is x
