"""CPU ORACLE -- test infrastructure only. NOT the product path.

A numpy restatement of the reference algorithms on the NEGF+GW hot path
(arxiv 2508.19138 restatement package ``negfgw``, mounted read-only at
/root/reference/pkg/src/negfgw). Each function cites the reference lines it
restates. Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
CPU-baseline leg may import this module, and only as the checker / the timed
CPU baseline -- the GPU product path never routes through it.

Parity pin: every function here is checked against golden vectors produced
by running the reference itself (tests/golden/make_golden.py, committed
fixtures tests/golden/*.npz) in tests/test_oracle_golden.py.

Layout: batched over energies. Diagonal blocks (n_e, n_b, bs, bs), off-diagonal
blocks (n_e, n_b-1, bs, bs), complex128. lg-compressed sources keep the
diagonal and upper blocks; B[i+1, i] = -B[i, i+1]^dag (blocks.py:110-118).
"""

from __future__ import annotations

import numpy as np
import scipy.linalg as sla
from scipy.fft import fft, ifft, next_fast_len
from scipy.special import expit


def _h(x: np.ndarray) -> np.ndarray:
    """Conjugate transpose of the trailing two axes."""
    return np.conj(np.swapaxes(x, -1, -2))


class OracleSingular(Exception):
    pass


def lu_inverse(a: np.ndarray) -> tuple[np.ndarray, float]:
    """_linalg.invert (_linalg.py:30-52): scipy LU + solve against I; raise on
    an exact-zero / non-finite pivot; return the pivot spread."""
    lu, piv = sla.lu_factor(a, check_finite=False)
    d = np.abs(np.diag(lu))
    if d.min() == 0.0 or not np.isfinite(d).all():
        raise OracleSingular("singular pivot")
    inv = sla.lu_solve((lu, piv), np.eye(a.shape[0], dtype=complex), check_finite=False)
    return inv, float(d.max() / d.min())


def _inv_batch(s: np.ndarray, step: int) -> np.ndarray:
    out = np.empty_like(s)
    for e in range(s.shape[0]):
        try:
            out[e], _ = lu_inverse(s[e])
        except (OracleSingular, ValueError, np.linalg.LinAlgError) as exc:
            raise OracleSingular(f"singular Schur complement at forward step {step}") from exc
    return out


# -- RGF selected solve ------------------------------------------------------


def rgf_forward(m_diag, m_up, m_lo, b_lg: dict | None = None):
    """forward_retarded (rgf.py:113-129) and forward_lg (rgf.py:132-149):
    returns (x_fwd list, {kind: xl_fwd list})."""
    b_lg = b_lg or {}
    n = m_diag.shape[1]
    # x_i = (M_ii - M_{i,i-1} x_{i-1} M_{i-1,i})^-1
    xf = [None] * n
    for i in range(n):
        s = m_diag[:, i]
        if i > 0:
            s = s - (m_lo[:, i - 1] @ xf[i - 1]) @ m_up[:, i - 1]
        xf[i] = _inv_batch(s, i)
    xlf = {}
    for kind, src in b_lg.items():
        bd, bu = src[0], src[1]
        xl = [None] * n
        for i in range(n):
            b = bd[:, i]
            if i > 0:
                a = m_lo[:, i - 1]
                y = (a @ xf[i - 1]) @ bu[:, i - 1]
                b = b + (a @ xl[i - 1]) @ _h(a) - (y - _h(y))
            xl[i] = (xf[i] @ b) @ _h(xf[i])
        xlf[kind] = xl
    return xf, xlf


def rgf_backward(m_diag, m_up, m_lo, b_lg: dict | None, xf, xlf, x_last=None, xl_last: dict | None = None,
                 symmetrize: bool = False) -> dict:
    """rgf_retarded (rgf.py:152-183) and rgf_lesser_greater (rgf.py:186-229)
    from the forward intermediates; ``x_last`` / ``xl_last`` seed the exact
    last diagonal blocks (as dist.py:692-697 does)."""
    b_lg = b_lg or {}
    n = m_diag.shape[1]
    out = {}
    xr_d = [None] * n
    xr_u = [None] * (n - 1)
    xr_l = [None] * (n - 1)
    xr_d[n - 1] = xf[n - 1] if x_last is None else x_last
    for i in range(n - 2, -1, -1):
        t = xf[i] @ m_up[:, i]
        u = t @ xr_d[i + 1]
        mx = m_lo[:, i] @ xf[i]
        xr_d[i] = xf[i] + u @ mx
        xr_u[i] = -u
        xr_l[i] = -(xr_d[i + 1] @ mx)
    out["xr_diag"] = np.stack(xr_d, 1)
    out["xr_upper"] = np.stack(xr_u, 1) if n > 1 else np.zeros_like(m_up)
    out["xr_lower"] = np.stack(xr_l, 1) if n > 1 else np.zeros_like(m_up)
    for kind, src in b_lg.items():
        bu = src[1]
        # explicit lower source blocks (FULL-storage sources, e.g. the W
        # system of scba.py:793-796); default: implied -B_{i,i+1}^dag
        bl = src[2] if len(src) > 2 else -_h(bu)
        xl = xlf[kind]
        d = [None] * n
        up = [None] * (n - 1)
        d[n - 1] = xl[n - 1] if xl_last is None else xl_last[kind]
        for i in range(n - 2, -1, -1):
            x = xf[i]
            t = x @ m_up[:, i]
            u = t @ xr_d[i + 1]
            y = (x @ bu[:, i]) @ _h(u)
            mxl = m_lo[:, i] @ xl[i]
            z = u @ mxl
            d[i] = xl[i] + (t @ d[i + 1]) @ _h(t) - (y - _h(y)) + (z - _h(z))
            b_dn = bl[:, i]  # B[i+1, i]
            lower = (xr_d[i + 1] @ b_dn) @ _h(x) - xr_d[i + 1] @ mxl - d[i + 1] @ _h(t)
            up[i] = -_h(lower)
        dd = np.stack(d, 1)
        if symmetrize:
            dd = 0.5 * (dd - _h(dd))
        out[f"x{kind}_diag"] = dd
        out[f"x{kind}_upper"] = np.stack(up, 1) if n > 1 else np.zeros_like(bu)
    return out


def rgf_selected(m_diag, m_up, m_lo, b_lg: dict | None = None, symmetrize: bool = False) -> dict:
    """Selected blocks of X^R = M^-1 and X^lg = M^-1 B^lg M^-dag.

    Restates rgf.py:113-129 (forward_retarded), rgf.py:132-149 (forward_lg),
    rgf.py:152-183 (rgf_retarded backward), rgf.py:186-229
    (rgf_lesser_greater backward) and rgf.py:82-88 (symmetrize), vectorised
    over the energy axis. ``b_lg`` maps kind ('<', '>') to (diag, upper).
    """
    xf, xlf = rgf_forward(m_diag, m_up, m_lo, b_lg)
    return rgf_backward(m_diag, m_up, m_lo, b_lg, xf, xlf, symmetrize=symmetrize)


# -- spatial domain decomposition (dist.py:69-717), partitions run in turn ----


def make_partition_plan(n_blocks: int, p_s: int) -> list[tuple[int, int]]:
    """dist.py:104-127: balanced contiguous ranges, leftovers to the middles."""
    if p_s < 1 or (p_s > 1 and n_blocks < 2 * p_s):
        raise ValueError(f"{n_blocks} blocks cannot feed {p_s} partitions of >= 2 blocks")
    base, rem = divmod(n_blocks, p_s)
    widths = [base] * p_s
    middles = list(range(1, p_s - 1)) or [0]
    order = middles + [r for r in range(p_s) if r not in middles]
    for k in range(rem):
        widths[order[k % len(order)]] += 1
    ranges, start = [], 0
    for w in widths:
        ranges.append((start, start + w - 1))
        start += w
    return ranges


def reverse_chain(md, mu, ml):
    """blocks.py reverse_blocks for a full-storage tridiagonal chain."""
    return md[:, ::-1].copy(), ml[:, ::-1].copy(), mu[:, ::-1].copy()


def reverse_lg(bd, bu):
    """reverse_blocks for lg-compressed sources: B_rev[t, t+1] = B[w-1-t, w-2-t] = -B[w-2-t, w-1-t]^dag."""
    return bd[:, ::-1].copy(), -_h(bu[:, ::-1])


def schur_tail(md, mu, ml, b_lg, xf, xlf):
    """dist.py:365-385: Schur complement and effective source at the last
    block after the forward elimination of the blocks before it."""
    last = md.shape[1] - 1
    a = ml[:, last - 1]
    t = a @ xf[last - 1]
    s = md[:, last] - t @ mu[:, last - 1]
    b_out = {}
    for k, (bd, bu) in b_lg.items():
        y = t @ bu[:, last - 1]
        b_out[k] = bd[:, last] + (a @ xlf[k][last - 1]) @ _h(a) - (y - _h(y))
    return s, b_out


def middle_sweep(md, mu, ml, b_lg):
    """dist.py:388-448: two-sided Schur elimination of interior blocks
    1..w-2; returns the 2x2 corner system and its sources per kind."""
    w = md.shape[1]
    kinds = list(b_lg)
    s_a = md[:, 0]
    b_a = {k: b_lg[k][0][:, 0] for k in kinds}
    if w == 2:
        return {"s_aa": s_a, "s_ab": mu[:, 0], "s_ba": ml[:, 0], "s_bb": md[:, 1], "b_aa": b_a,
                "b_ab": {k: b_lg[k][1][:, 0] for k in kinds}, "b_bb": {k: b_lg[k][0][:, 1] for k in kinds}}
    f, f_p, s_i = mu[:, 0], ml[:, 0], md[:, 1]
    b_ai = {k: b_lg[k][1][:, 0] for k in kinds}
    b_i = {k: b_lg[k][0][:, 1] for k in kinds}
    for i in range(1, w - 1):
        y = _inv_batch(s_i, i)
        fy = f @ y
        m_dn, m_up = ml[:, i], mu[:, i]
        my = m_dn @ y
        s_a = s_a - fy @ f_p
        for k in kinds:
            bd, bu = b_lg[k]
            ybh = (y @ b_i[k]) @ _h(y)
            fyb = f @ ybh
            myb = m_dn @ ybh
            t1 = my @ bu[:, i]
            b_a[k] = b_a[k] + fy @ _h(b_ai[k]) - b_ai[k] @ _h(fy) + fyb @ _h(f)
            b_ai[k] = -(fy @ bu[:, i]) - b_ai[k] @ _h(my) + fyb @ _h(m_dn)
            b_i[k] = bd[:, i + 1] - t1 + _h(t1) + myb @ _h(m_dn)
        f, f_p = -(fy @ m_up), -(my @ f_p)
        s_i = md[:, i + 1] - my @ m_up
    return {"s_aa": s_a, "s_ab": f, "s_ba": f_p, "s_bb": s_i, "b_aa": b_a, "b_ab": b_ai, "b_bb": b_i}


def fold_corner(md, b_lg, j, m_out, m_in, b_out, b_in, x_env, xl_env):
    """dist.py:451-473 (in place on md and the source diagonals)."""
    t = m_out @ x_env
    md[:, j] = md[:, j] - t @ m_in
    for k, (bd, _bu) in b_lg.items():
        bd[:, j] = bd[:, j] + (-(t @ b_in[k]) - (b_out[k] @ _h(x_env)) @ _h(m_out) + (m_out @ xl_env[k]) @ _h(m_out))


def dd_selected(m_diag, m_up, m_lo, b_lg: dict, ranges) -> dict:
    """dist_selected_solve (dist.py:622-717) with the partitions of ``ranges``
    executed one after another: local eliminations (ends: forward sweep +
    Schur tail, the bottom on the reversed chain; middles: two-sided sweep),
    the reduced boundary chain (dist.py:486-561), then local recovery (ends:
    backward sweep seeded with the exact boundary block; middles: corner
    folds + local selected solve) and assembly (dist.py:587-619)."""
    p_s = len(ranges)
    if p_s == 1:
        return rgf_selected(m_diag, m_up, m_lo, b_lg)
    n = m_diag.shape[1]
    kinds = list(b_lg)
    loc, contribs = [], []
    for r, (a, b) in enumerate(ranges):
        if r == 0 or r == p_s - 1:
            lo_, hi_ = (0, b) if r == 0 else (a, n - 1)
            md, mu, ml = m_diag[:, lo_:hi_ + 1].copy(), m_up[:, lo_:hi_].copy(), m_lo[:, lo_:hi_].copy()
            bl = {k: (b_lg[k][0][:, lo_:hi_ + 1].copy(), b_lg[k][1][:, lo_:hi_].copy()) for k in kinds}
            if r == p_s - 1:
                md, mu, ml = reverse_chain(md, mu, ml)
                bl = {k: reverse_lg(*bl[k]) for k in kinds}
            xf, xlf = rgf_forward(md, mu, ml, bl)
            contribs.append(schur_tail(md, mu, ml, bl, xf, xlf))
            loc.append((md, mu, ml, bl, xf, xlf))
        else:
            md, mu, ml = m_diag[:, a:b + 1].copy(), m_up[:, a:b].copy(), m_lo[:, a:b].copy()
            bl = {k: (b_lg[k][0][:, a:b + 1].copy(), b_lg[k][1][:, a:b].copy()) for k in kinds}
            contribs.append(middle_sweep(md, mu, ml, bl))
            loc.append((md, mu, ml, bl, None, None))
    # reduced chain over the boundary nodes
    nodes = [ranges[0][1]] + [x for a, b in ranges[1:-1] for x in (a, b)] + [ranges[-1][0]]
    nr = len(nodes)
    ne, bs = m_diag.shape[0], m_diag.shape[-1]
    z = lambda k: np.zeros((ne, k, bs, bs), complex)
    rd, ru, rl = z(nr), z(nr - 1), z(nr - 1)
    rb = {k: (z(nr), z(nr - 1)) for k in kinds}
    s_top, b_top = contribs[0]
    rd[:, 0] = s_top
    for k in kinds:
        rb[k][0][:, 0] = b_top[k]
    for j in range(1, p_s - 1):
        sw, p0, p1 = contribs[j], 2 * j - 1, 2 * j
        rd[:, p0], rd[:, p1], ru[:, p0], rl[:, p0] = sw["s_aa"], sw["s_bb"], sw["s_ab"], sw["s_ba"]
        for k in kinds:
            rb[k][0][:, p0], rb[k][0][:, p1], rb[k][1][:, p0] = sw["b_aa"][k], sw["b_bb"][k], sw["b_ab"][k]
    s_bot, b_bot = contribs[-1]
    rd[:, nr - 1] = s_bot
    for k in kinds:
        rb[k][0][:, nr - 1] = b_bot[k]
    for p0 in range(0, nr - 1, 2):
        g = nodes[p0]
        ru[:, p0], rl[:, p0] = m_up[:, g], m_lo[:, g]
        for k in kinds:
            rb[k][1][:, p0] = b_lg[k][1][:, g]
    xf_r, xlf_r = rgf_forward(rd, ru, rl, rb)
    sol_r = rgf_backward(rd, ru, rl, rb, xf_r, xlf_r)
    rvd, rvu, rvl = reverse_chain(rd, ru, rl)
    xf_v, xlf_v = rgf_forward(rvd, rvu, rvl, {k: reverse_lg(*rb[k]) for k in kinds})
    out = {"xr_diag": np.zeros_like(m_diag), "xr_upper": np.zeros_like(m_up), "xr_lower": np.zeros_like(m_up)}
    for k in kinds:
        out[f"x{k}_diag"] = np.zeros_like(m_diag)
        out[f"x{k}_upper"] = np.zeros_like(m_up)
    for r, (a, b) in enumerate(ranges):
        md, mu, ml, bl, xf, xlf = loc[r]
        w = b - a + 1
        if r == 0 or r == p_s - 1:
            node = 0 if r == 0 else nr - 1
            sol = rgf_backward(md, mu, ml, bl, xf, xlf, x_last=sol_r["xr_diag"][:, node],
                               xl_last={k: sol_r[f"x{k}_diag"][:, node] for k in kinds})
            if r == p_s - 1:  # back to global order (dist.py:564-584)
                sol = {"xr_diag": sol["xr_diag"][:, ::-1], "xr_upper": sol["xr_lower"][:, ::-1],
                       "xr_lower": sol["xr_upper"][:, ::-1],
                       **{f"x{k}_diag": sol[f"x{k}_diag"][:, ::-1] for k in kinds},
                       **{f"x{k}_upper": -_h(sol[f"x{k}_upper"][:, ::-1]) for k in kinds}}
        else:
            left, right = 2 * r - 2, nr - 1 - (2 * r + 1)
            fold_corner(md, bl, 0, m_lo[:, a - 1], m_up[:, a - 1], {k: -_h(b_lg[k][1][:, a - 1]) for k in kinds},
                        {k: b_lg[k][1][:, a - 1] for k in kinds}, xf_r[left], {k: xlf_r[k][left] for k in kinds})
            fold_corner(md, bl, w - 1, m_up[:, b], m_lo[:, b], {k: b_lg[k][1][:, b] for k in kinds},
                        {k: -_h(b_lg[k][1][:, b]) for k in kinds}, xf_v[right], {k: xlf_v[k][right] for k in kinds})
            sol = rgf_selected(md, mu, ml, bl)
        out["xr_diag"][:, a:b + 1] = sol["xr_diag"]
        out["xr_upper"][:, a:b] = sol["xr_upper"]
        out["xr_lower"][:, a:b] = sol["xr_lower"]
        for k in kinds:
            out[f"x{k}_diag"][:, a:b + 1] = sol[f"x{k}_diag"]
            out[f"x{k}_upper"][:, a:b] = sol[f"x{k}_upper"]
    for p0 in range(0, nr - 1, 2):  # cross-partition blocks from the reduced solve
        g = nodes[p0]
        out["xr_upper"][:, g], out["xr_lower"][:, g] = sol_r["xr_upper"][:, p0], sol_r["xr_lower"][:, p0]
        for k in kinds:
            out[f"x{k}_upper"][:, g] = sol_r[f"x{k}_upper"][:, p0]
    return out


def to_dense(diag, up, lo) -> np.ndarray:
    """Block-tridiagonal (single energy) to a dense matrix."""
    n, bs = diag.shape[0], diag.shape[1]
    a = np.zeros((n * bs, n * bs), dtype=complex)
    for i in range(n):
        a[i * bs:(i + 1) * bs, i * bs:(i + 1) * bs] = diag[i]
        if i + 1 < n:
            a[i * bs:(i + 1) * bs, (i + 1) * bs:(i + 2) * bs] = up[i]
            a[(i + 1) * bs:(i + 2) * bs, i * bs:(i + 1) * bs] = lo[i]
    return a


def dense_selected(m_diag, m_up, m_lo, b_lg: dict | None = None) -> dict:
    """rgf.py:246-267 dense_selected_oracle: full inverse + triple product."""
    b_lg = b_lg or {}
    ne, n, bs = m_diag.shape[:3]
    out = {k: [] for k in ("xr_diag", "xr_upper", "xr_lower")}
    for kind in b_lg:
        out[f"x{kind}_diag"] = []
        out[f"x{kind}_upper"] = []
    cut = lambda d, i, j: d[i * bs:(i + 1) * bs, j * bs:(j + 1) * bs]
    for e in range(ne):
        g = np.linalg.inv(to_dense(m_diag[e], m_up[e], m_lo[e]))
        out["xr_diag"].append([cut(g, i, i) for i in range(n)])
        out["xr_upper"].append([cut(g, i, i + 1) for i in range(n - 1)])
        out["xr_lower"].append([cut(g, i + 1, i) for i in range(n - 1)])
        for kind, (bd, bu) in b_lg.items():
            bf = to_dense(bd[e], bu[e], -_h(bu[e]))
            f = g @ bf @ g.conj().T
            out[f"x{kind}_diag"].append([cut(f, i, i) for i in range(n)])
            out[f"x{kind}_upper"].append([cut(f, i, i + 1) for i in range(n - 1)])
    return {k: np.asarray(v).reshape((ne, -1, bs, bs)) for k, v in out.items()}


# -- seeded inputs (toys.py) -------------------------------------------------


def random_bt_system(seed: int, n_blocks: int | None = None, block_size: int | None = None,
                     max_blocks: int = 10, max_block_size: int = 8):
    """toys.py:33-65: same RNG draw order, returned as stacked arrays
    (m_diag, m_up, m_lo, {'<': (d, u), '>': (d, u)}) with a leading n_e=1 axis."""
    rng = np.random.default_rng(seed)
    n = int(n_blocks or rng.integers(2, max_blocks + 1))
    bs = int(block_size or rng.integers(1, max_block_size + 1))
    rb = lambda: rng.standard_normal((bs, bs)) + 1j * rng.standard_normal((bs, bs))
    md = np.zeros((n, bs, bs), complex)
    mu = np.zeros((n - 1, bs, bs), complex)
    ml = np.zeros((n - 1, bs, bs), complex)
    for i in range(n):
        md[i] = rb() + (4.0 + 1.0j) * np.eye(bs)
        if i + 1 < n:
            mu[i] = 0.5 * rb()
            ml[i] = 0.5 * rb()
    src = []
    for _ in range(2):
        bd = np.zeros((n, bs, bs), complex)
        bu = np.zeros((n - 1, bs, bs), complex)
        for i in range(n):
            d = rb()
            bd[i] = 0.5 * (d - d.conj().T)
            if i + 1 < n:
                bu[i] = rb()
        src.append((bd[None], bu[None]))
    return md[None], mu[None], ml[None], {"<": src[0], ">": src[1]}


def chain_device(n_blocks: int, block_size: int, t: float = 0.4, onsite_seed: int = 7,
                 onsite_scale: float = 0.15):
    """toys.py:89-108: (h_diag, h_upper, h_lower) of the homogeneous chain."""
    rng = np.random.default_rng(onsite_seed)
    a = rng.standard_normal((block_size,) * 2) + 1j * rng.standard_normal((block_size,) * 2)
    onsite = onsite_scale * 0.5 * (a + a.conj().T)
    c = t * np.eye(block_size, dtype=complex) + 0.05 * (
        rng.standard_normal((block_size,) * 2) + 1j * rng.standard_normal((block_size,) * 2))
    hd = np.broadcast_to(onsite, (n_blocks, block_size, block_size)).copy()
    hu = np.broadcast_to(c, (n_blocks - 1, block_size, block_size)).copy()
    hl = np.broadcast_to(c.conj().T, (n_blocks - 1, block_size, block_size)).copy()
    return hd, hu, hl


def coulomb_matrix(n_blocks: int, block_size: int, v0: float = 1e-3, seed: int = 11):
    """toys.py:111-132: real symmetric replicated interaction (diag, up, lo)."""
    rng = np.random.default_rng(seed)
    d = rng.standard_normal((block_size, block_size))
    diag = v0 * (np.eye(block_size) + 0.1 * (d + d.T))
    off = v0 * 0.3 * rng.standard_normal((block_size, block_size))
    vd = np.broadcast_to(diag.astype(complex), (n_blocks, block_size, block_size)).copy()
    vu = np.broadcast_to(off.astype(complex), (n_blocks - 1, block_size, block_size)).copy()
    vl = np.broadcast_to(off.T.astype(complex), (n_blocks - 1, block_size, block_size)).copy()
    return vd, vu, vl


def fermi(e, mu, kT):
    """device.py:32-36."""
    return expit(-(np.asarray(e, dtype=float) - mu) / kT)


# -- open boundary conditions (obc.py) ----------------------------------------


class OracleConvergence(Exception):
    pass


def recursion_residual(m, n, n_prime, x) -> float:
    """obc.py:98-104: relative defect of x = (m - n x n')^-1."""
    lhs, _ = lu_inverse(m - (n @ x) @ n_prime)
    num, den = np.linalg.norm(lhs - x), np.linalg.norm(x)
    return float(num / den) if den > 0 else float(num)


def sancho_rubio(m, n, n_prime, tol: float = 1e-12, max_iter: int = 100):
    """obc.py:144-182 decimation; returns (x, sweeps, residual)."""
    s, b, al, be = m.copy(), m.copy(), n.copy(), n_prime.copy()
    scale = max(np.linalg.norm(n), np.linalg.norm(n_prime), 1e-300)
    for it in range(1, max_iter + 1):
        g, _ = lu_inverse(b)
        ag, bg = al @ g, be @ g
        agb, bga = ag @ be, bg @ al
        s = s - agb
        b = b - agb - bga
        al, be = ag @ al, bg @ be
        if np.linalg.norm(al) + np.linalg.norm(be) < tol * scale:
            x, _ = lu_inverse(s)
            res = recursion_residual(m, n, n_prime, x)
            if not np.isfinite(res) or res > 10 * max(tol, 1e-14):
                raise OracleConvergence(f"residual {res:.3e}")
            return x, it, res
    raise OracleConvergence("not converged")


BEYN_PROBE_SEED = 1278  # obc.py:47


def beyn(m, n, n_prime, n_quad: int = 16, radius: float = 1.0, center: complex = 0.0, svd_tol: float = 1e-8,
         probe_seed: int = BEYN_PROBE_SEED):
    """obc_beyn (obc.py:198-296) for a nearest-neighbour lead (stencil
    [n', m, n], N_U = 1): contour moments of P(z)^-1 = (n' + z m + z^2 n)^-1
    against a seeded probe, rank-revealing SVD, the small eigenproblem, the
    decaying modes |mu| < 1 - 1e-8, then x = (m + n F)^-1 with
    F = Phi diag(mu) Phi^+. Returns (x, n_modes)."""
    bs = m.shape[0]
    if np.allclose(n, 0):
        return lu_inverse(m)[0], 0
    rng = np.random.default_rng(probe_seed)
    probe = rng.standard_normal((bs, bs)) + 1j * rng.standard_normal((bs, bs))
    a0 = np.zeros((bs, bs), complex)
    a1 = np.zeros((bs, bs), complex)
    for k in range(n_quad):
        z = center + radius * np.exp(2j * np.pi * k / n_quad)
        pz = n_prime + z * m + z * z * n
        rz = sla.lu_solve(sla.lu_factor(pz, check_finite=False), probe, check_finite=False)
        w = (z - center) / n_quad
        a0 += w * rz
        a1 += w * z * rz
    u, sig, wh = np.linalg.svd(a0)
    rank = int(np.sum(sig > svd_tol * sig[0])) if sig[0] > 0 else 0
    if rank == 0:
        return lu_inverse(m)[0], 0
    u = u[:, :rank]
    w_red = wh.conj().T[:, :rank]
    b_small = (u.conj().T @ a1 @ w_red) / sig[:rank]
    mu, vecs = np.linalg.eig(b_small)
    keep = np.abs(mu) < 1.0 - 1e-8
    mu, vecs = mu[keep], vecs[:, keep]
    if mu.size == 0:
        return lu_inverse(m)[0], 0
    phi = u @ vecs
    f_mat = (phi * mu[None, :]) @ np.linalg.pinv(phi)
    return lu_inverse(m + n @ f_mat)[0], int(mu.size)


def sigma_lg_obc(x_r, mu, kT, energy, n, n_prime):
    """obc.py:460-486."""
    sr = (n @ x_r) @ n_prime
    gam = sr - _h(sr)
    f = float(fermi(energy, mu, kT))
    return sr, -f * gam, (1.0 - f) * gam


def spectral_radius_estimate(a, n_iter: int = 50, seed: int = 5) -> float:
    """obc.py:320-342 power iteration."""
    rng = np.random.default_rng(seed)
    v = rng.standard_normal(a.shape[0]) + 1j * rng.standard_normal(a.shape[0])
    v /= np.linalg.norm(v)
    rho = 0.0
    for _ in range(n_iter):
        w = a @ v
        nw = np.linalg.norm(w)
        if nw == 0:
            return 0.0
        rho, v = nw, w / nw
    return float(rho)


def stein_geometric(a, q, tol: float = 1e-12, max_iter: int = 100):
    """obc.py:427-447: w - a w a^dag = q by squared doubling."""
    if spectral_radius_estimate(a) >= 1.0:
        raise OracleConvergence("spectral radius >= 1")
    w, ak = q.copy(), a.copy()
    for _ in range(max_iter):
        upd = (ak @ w) @ _h(ak)
        w = w + upd
        if np.linalg.norm(upd) < tol * max(np.linalg.norm(w), 1e-300):
            return w
        ak = ak @ ak
    raise OracleConvergence("stein not converged")


def stein_direct(a, q):
    """scba.py:534-543: doubling with the dense vectorised fallback."""
    try:
        return stein_geometric(a, q)
    except OracleConvergence:
        n = a.shape[0]
        lhs = np.eye(n * n, dtype=complex) - np.kron(a.conj(), a)
        return np.linalg.solve(lhs, q.ravel(order="F")).reshape((n, n), order="F")


# -- runtime memoization (obc.py:490-608) --------------------------------------


class SurfaceCache:
    """obc.py:498-515: cached surface blocks keyed by (subsystem, side,
    energy index, kind) plus direct/memoized call counters."""

    def __init__(self, n_fpi_retarded: int = 20, n_fpi_lg: int = 10) -> None:
        self.n_fpi_retarded, self.n_fpi_lg = n_fpi_retarded, n_fpi_lg
        self.entries: dict = {}
        self.stats = {"direct_calls": 0, "memoized_calls": 0}

    def n_fpi(self, kind: str) -> int:
        return self.n_fpi_retarded if kind == "R" else self.n_fpi_lg


def fixed_point_step(m, n, n_prime, x):
    """obc.py:138-141: x <- (m - n x n')^-1 (raises OracleSingular)."""
    inv, _ = lu_inverse(m - (n @ x) @ n_prime)
    return inv


def _memo_direct(key, direct, cache):
    """obc.py:603-608."""
    x = direct()
    cache.entries[key] = np.asarray(x)
    cache.stats["direct_calls"] += 1
    return x


def _memo_accept(key, x, cache):
    cache.entries[key] = x
    cache.stats["memoized_calls"] += 1
    return x


def memoized_obc(key, direct, iterative, cache: SurfaceCache, n_fpi: int, tol: float):
    """obc.py:519-600: two trial fixed-point updates from the cached block give
    the update size and a contraction estimate rho; refresh with the budget
    n_fpi only when the budgeted tail delta2 rho^(n_fpi-2) rho/(1-rho) < tol,
    stop early once the tail bound is below tol, else solve directly. Any
    non-finite iterate or singular update falls back to the direct solver."""
    x0 = cache.entries.get(key)
    if x0 is None:
        return _memo_direct(key, direct, cache)
    try:
        with np.errstate(over="ignore", invalid="ignore"):
            x1 = iterative(x0)
            d1, s1 = np.linalg.norm(x1 - x0), np.linalg.norm(x1)
            if not np.isfinite(d1) or s1 == 0 or not np.all(np.isfinite(x1)):
                return _memo_direct(key, direct, cache)
            delta1 = d1 / s1
            if delta1 == 0.0:
                return _memo_accept(key, x1, cache)
            x2 = iterative(x1)
            d2, s2 = np.linalg.norm(x2 - x1), np.linalg.norm(x2)
            if not np.isfinite(d2) or s2 == 0 or not np.all(np.isfinite(x2)):
                return _memo_direct(key, direct, cache)
            delta2 = d2 / s2
            if delta2 <= 1e-14:
                return _memo_accept(key, x2, cache)
            rho = delta2 / delta1
            if rho >= 1.0:
                return _memo_direct(key, direct, cache)
            tail = rho / (1.0 - rho)
            if delta2 * rho ** max(0, n_fpi - 2) * tail >= tol:
                return _memo_direct(key, direct, cache)
            x, last = x2, delta2
            for _ in range(max(0, n_fpi - 2)):
                if last * tail < tol:
                    break
                x_new = iterative(x)
                if not np.all(np.isfinite(x_new)):
                    return _memo_direct(key, direct, cache)
                last = np.linalg.norm(x_new - x) / max(np.linalg.norm(x_new), 1e-300)
                x = x_new
            if last * tail >= tol:
                return _memo_direct(key, direct, cache)
            return _memo_accept(key, x, cache)
    except (OracleSingular, OracleConvergence, ValueError, np.linalg.LinAlgError):
        return _memo_direct(key, direct, cache)


# -- carrier system (scba.py:670-775) ------------------------------------------


def assemble_g(energies, eta, h, f_bath, sr=None, sl=None, sg=None):
    """scba.py:670-727 for a batch of energies. h = (diag, up, lo) of H;
    sr = (diag, up, lo) of Sigma^R_scatt, sl/sg = (diag, up) of Sigma^<>_scatt
    (all energy-major), any may be None. Returns m=(d,u,l), bl=(d,u), bg=(d,u)."""
    hd, hu, hl = h
    ne, bs = len(energies), hd.shape[-1]
    eye = np.eye(bs)
    z = (np.asarray(energies) + 1j * eta)[:, None, None, None]
    md = z * eye - hd[None]
    mu = np.broadcast_to(-hu[None], (ne,) + hu.shape).copy()
    ml = np.broadcast_to(-hl[None], (ne,) + hl.shape).copy()
    if sr is not None:
        md, mu, ml = md - sr[0], mu - sr[1], ml - sr[2]
    f = np.asarray(f_bath)[:, None, None, None]
    bld = np.broadcast_to((2j * eta * f) * eye, md.shape) + (0 if sl is None else sl[0])
    bgd = np.broadcast_to((-2j * eta * (1.0 - f)) * eye, md.shape) + (0 if sg is None else sg[0])
    blu = np.zeros_like(mu) if sl is None else sl[1].copy()
    bgu = np.zeros_like(mu) if sg is None else sg[1].copy()
    return (md, mu, ml), (np.ascontiguousarray(bld), blu), (np.ascontiguousarray(bgd), bgu)


def g_closure(m, bl, bg, energies, mu_left, mu_right, kT, tol, cache: SurfaceCache | None = None,
              tol_memo: float = 0.0):
    """scba.py:755-774: per side, Sancho on the contact cell (_lead_cell,
    scba.py:558-574), sigma_lg_obc, corner updates. In place; returns the
    boundary lesser/greater self-energies {side: (sl, sg)} (n_e, bs, bs).
    With ``cache`` the surface goes through memoized_obc (scba.py:577-614)."""
    md, mu, ml = m
    n_b = md.shape[1]
    out = {}
    for side, mu_c in (("left", mu_left), ("right", mu_right)):
        c = 0 if side == "left" else n_b - 1
        sls, sgs = [], []
        for e, E in enumerate(energies):
            if side == "left":
                cell = (md[e, 0], ml[e, 0], mu[e, 0])
            else:
                cell = (md[e, n_b - 1], mu[e, n_b - 2], ml[e, n_b - 2])
            x = _surface(cell, "G", side, e, tol, cache, tol_memo)
            sr, s_l, s_g = sigma_lg_obc(x, mu_c, kT, E, cell[1], cell[2])
            md[e, c] = md[e, c] - sr
            bl[0][e, c] = bl[0][e, c] + s_l
            bg[0][e, c] = bg[0][e, c] + s_g
            sls.append(s_l)
            sgs.append(s_g)
        out[side] = (np.stack(sls), np.stack(sgs))
    return out


def _surface(cell, subsystem, side, e, tol, cache, tol_memo):
    """_retarded_surface (scba.py:577-614) with the Sancho direct solver."""
    direct = lambda: sancho_rubio(*cell, tol=tol)[0]
    if cache is None:
        return direct()
    return memoized_obc((subsystem, side, e, "R"), direct, lambda x: fixed_point_step(*cell, x), cache,
                        cache.n_fpi("R"), tol_memo)


def ballistic(h, energies, eta, mu_left, mu_right, kT, tol=1e-8):
    """scba_run with v_mat=None, retarded_method='sancho', memoizer off
    (scba.py:951-1011): one carrier solve per energy, symmetrized."""
    f_bath = fermi(energies, 0.5 * (mu_left + mu_right), kT)
    m, bl, bg = assemble_g(energies, eta, h, f_bath)
    obc = g_closure(m, bl, bg, energies, mu_left, mu_right, kT, tol)
    sol = rgf_selected(*m, {"<": bl, ">": bg}, symmetrize=True)
    return {
        "g_r_diag": sol["xr_diag"], "g_r_upper": sol["xr_upper"], "g_r_lower": sol["xr_lower"],
        "g_lesser_diag": sol["x<_diag"], "g_lesser_upper": sol["x<_upper"],
        "g_greater_diag": sol["x>_diag"], "g_greater_upper": sol["x>_upper"],
        "sigma_obc_lesser_left": obc["left"][0], "sigma_obc_greater_left": obc["left"][1],
        "sigma_obc_lesser_right": obc["right"][0], "sigma_obc_greater_right": obc["right"][1],
    }


def observables(res: dict, h_upper, de: float) -> dict:
    """scba.py:1313-1376: dos, electron_density, current_spectrum,
    terminal_current for result arrays named like ScbaResult fields."""
    c_obs = 1.0 / (2.0 * np.pi)
    tr_r = np.trace(res["g_r_diag"], axis1=2, axis2=3)
    tr_l = np.trace(res["g_lesser_diag"], axis1=2, axis2=3)
    n_b = res["g_r_diag"].shape[1]
    cur = np.zeros((tr_r.shape[0], n_b - 1))
    for i in range(n_b - 1):
        gl_lower = -np.conj(np.swapaxes(res["g_lesser_upper"][:, i], 1, 2))
        cur[:, i] = c_obs * 2.0 * np.einsum("ij,eji->e", h_upper[i], gl_lower).real

    def term(sl, sg, c):
        tr = np.einsum("eij,eji->e", sl, res["g_greater_diag"][:, c]) - np.einsum(
            "eij,eji->e", sg, res["g_lesser_diag"][:, c])
        return float(c_obs * de * tr.real.sum())

    return {
        "dos": -tr_r.imag / np.pi,
        "density": (c_obs * de * (-1j * tr_l).sum(axis=0)).real,
        "current_spectrum": cur,
        "terminal_left": term(res["sigma_obc_lesser_left"], res["sigma_obc_greater_left"], 0),
        "terminal_right": term(res["sigma_obc_lesser_right"], res["sigma_obc_greater_right"], n_b - 1),
    }


# -- energy convolutions (convolve.py) ------------------------------------------


def convolve_energy(x1, x2, mode, prefactor, de):
    """convolve.py:39-71: FFT linear convolution / correlation, window, scale."""
    x1 = np.asarray(x1, dtype=complex)
    x2 = np.asarray(x2, dtype=complex)
    n = x1.shape[-1]
    if mode == "correlation":
        x2 = x2[..., ::-1]
    m = next_fast_len(2 * n - 1)
    full = ifft(fft(x1, n=m) * fft(x2, n=m), n=m)
    out = full[..., n - 1:2 * n - 1] if mode == "correlation" else full[..., :n]
    return prefactor * de * out


def convolve_energy_direct(x1, x2, mode, prefactor, de):
    """convolve.py:74-98: O(N^2) sum (vectorised over the lag)."""
    n = x1.shape[-1]
    out = np.zeros(np.broadcast(x1, x2).shape, dtype=complex)
    for k in range(n):
        if mode == "convolution":
            out[..., k] = np.sum(x1[..., k::-1] * x2[..., :k + 1], axis=-1)
        else:
            out[..., k] = np.sum(x1[..., k:] * x2[..., :n - k], axis=-1)
    return prefactor * de * out


def retarded_from_lg(xl, xg):
    """convolve.py:101-129: r = ifft(theta * fft(xg - xl, m))[:N]."""
    n = xl.shape[-1]
    m = next_fast_len(2 * n)
    if m % 2 == 1:
        m = next_fast_len(m + 1)
    theta = np.zeros(m)
    theta[0] = theta[m // 2] = 0.5
    theta[1:m // 2] = 1.0
    return ifft(theta * fft(xg - xl, n=m), n=m)[..., :n]


def project_diag_rows(arr, diag_mask):
    """scba.py:406-409."""
    arr = arr.copy()
    arr[diag_mask] = 0.5 * (arr[diag_mask] - np.conj(arr[diag_mask]))
    return arr


def polarization(gl, gg, diag_mask, de, c=-1j / (2.0 * np.pi)):
    """scba.py:1035-1048."""
    pl = project_diag_rows(convolve_energy(gl, -np.conj(gg), "correlation", c, de), diag_mask)
    pg = project_diag_rows(convolve_energy(gg, -np.conj(gl), "correlation", c, de), diag_mask)
    return pl, pg, retarded_from_lg(pl, pg), retarded_from_lg(-np.conj(pl), -np.conj(pg))


def self_energy(gl, gg, wl, wg, diag_mask, de, c=1j / (2.0 * np.pi)):
    """scba.py:1118-1132 (W rows already gathered onto the G pattern)."""
    sl = project_diag_rows(convolve_energy(gl, wl, "convolution", c, de), diag_mask)
    sg = project_diag_rows(convolve_energy(gg, wg, "convolution", c, de), diag_mask)
    return sl, sg, retarded_from_lg(sl, sg), retarded_from_lg(-np.conj(sl), -np.conj(sg))


# -- entry-major layout (convolve.py:135-187, scba.py:252-325) ------------------


def entry_pattern(n_b: int, bs: int):
    """Compressed bandwidth-3 EntryPattern: (rows, cols) global indices."""
    r, c = np.triu_indices(bs)
    rows, cols = [], []
    for bi in range(n_b):
        rows.append(bi * bs + r)
        cols.append(bi * bs + c)
        if bi + 1 < n_b:
            rr, cc = np.divmod(np.arange(bs * bs), bs)
            rows.append(bi * bs + rr)
            cols.append((bi + 1) * bs + cc)
    return np.concatenate(rows), np.concatenate(cols)


def gather_entries(diag, upper):
    """_gather_entries for a batch: (ne, n_b, bs, bs) + (ne, n_b-1, bs, bs) -> (n_entries, ne)."""
    ne, n_b, bs = diag.shape[:3]
    r, c = np.triu_indices(bs)
    parts = []
    for bi in range(n_b):
        parts.append(diag[:, bi][:, r, c])
        if bi + 1 < n_b:
            parts.append(upper[:, bi].reshape(ne, bs * bs))
    return np.concatenate(parts, axis=1).T.copy()


def scatter_lg(values, n_b, bs):
    """_scatter_lg: (n_entries, ne) -> diag (mirror rule), upper."""
    ne = values.shape[1]
    r, c = np.triu_indices(bs)
    t = len(r)
    d = np.zeros((ne, n_b, bs, bs), complex)
    u = np.zeros((ne, max(n_b - 1, 0), bs, bs), complex)
    k = 0
    off = r != c
    for bi in range(n_b):
        v = values[k:k + t].T
        d[:, bi][:, r, c] = v
        d[:, bi][:, c[off], r[off]] = -np.conj(v[:, off])
        k += t
        if bi + 1 < n_b:
            u[:, bi] = values[k:k + bs * bs].T.reshape(ne, bs, bs)
            k += bs * bs
    return d, u


def scatter_retarded(up, lo, n_b, bs):
    """_scatter_retarded: upper values at (r,c), lower values at (c,r)."""
    ne = up.shape[1]
    r, c = np.triu_indices(bs)
    t = len(r)
    d = np.zeros((ne, n_b, bs, bs), complex)
    u = np.zeros((ne, max(n_b - 1, 0), bs, bs), complex)
    l = np.zeros_like(u)
    k = 0
    for bi in range(n_b):
        d[:, bi][:, r, c] = up[k:k + t].T
        d[:, bi][:, c, r] = lo[k:k + t].T  # diagonal elements end with the lower value
        k += t
        if bi + 1 < n_b:
            u[:, bi] = up[k:k + bs * bs].T.reshape(ne, bs, bs)
            l[:, bi] = np.swapaxes(lo[k:k + bs * bs].T.reshape(ne, bs, bs), 1, 2)
            k += bs * bs
    return d, u, l


# -- screened interaction (scba.py:784-858) -------------------------------------


def _band_product(a, b):
    """Banded block product of two (d, u, l) tridiagonal batches, returned as a
    dict {(i, j): block batch} over the full product band (bt_multiply)."""
    ad, au, al = a
    bd, bu, bl = b
    n = ad.shape[1]

    def get(x, i, j):
        d, u, l = x
        if i == j:
            return d[:, i]
        if j == i + 1:
            return u[:, i]
        if i == j + 1:
            return l[:, j]
        return None

    out = {}
    for i in range(n):
        for j in range(max(0, i - 2), min(n, i + 3)):
            acc = None
            for k in range(max(0, i - 1, j - 1), min(n, i + 2, j + 2)):
                x, y = get(a, i, k), get(b, k, j)
                if x is None or y is None:
                    continue
                acc = x @ y if acc is None else acc + x @ y
            if acc is not None:
                out[(i, j)] = acc
    return out


def w_system(v, pr, pl, pg):
    """_w_lhs / _w_rhs (scba.py:784-796) for a batch. v = (d, u, l) energy
    independent; pr = (d, u, l); pl, pg = (d, u) lg-compressed. Returns
    m = (d, u, l) and full-storage sources {'<': (d, u, l), '>': (d, u, l)}."""
    ne = pr[0].shape[0]
    n = v[0].shape[0]
    vb = tuple(np.broadcast_to(x[None], (ne,) + x.shape) for x in v)
    vp = _band_product(vb, pr)
    eye = np.eye(v[0].shape[-1])
    md = np.stack([eye - vp[(i, i)] for i in range(n)], 1)
    mu = np.stack([-vp[(i, i + 1)] for i in range(n - 1)], 1)
    ml = np.stack([-vp[(i + 1, i)] for i in range(n - 1)], 1)
    srcs = {}
    for kind, (d, u) in (("<", pl), (">", pg)):
        p = (d, u, -_h(u))
        q = _band_product(vb, p)  # V P, bandwidth 5
        b = {}
        for i in range(n):
            for j in range(max(0, i - 1), min(n, i + 2)):
                acc = None
                for k in range(max(0, i - 2, j - 1), min(n, i + 3, j + 2)):
                    x = q.get((i, k))
                    if x is None:
                        continue
                    y = vb[0][:, k] if k == j else (vb[1][:, k] if j == k + 1 else vb[2][:, j])
                    acc = x @ y if acc is None else acc + x @ y
                b[(i, j)] = acc
        srcs[kind] = (np.stack([b[(i, i)] for i in range(n)], 1),
                      np.stack([b[(i, i + 1)] for i in range(n - 1)], 1),
                      np.stack([b[(i + 1, i)] for i in range(n - 1)], 1))
    return (md, mu, ml), srcs


def w_closure(m, srcs, surface_tol, cache: SurfaceCache | None = None, tol_memo: float = 0.0):
    """scba.py:839-858 + _lead_lg_boundary (:617-664), W surface by Sancho;
    with ``cache`` both the surface and the Stein solve are memoized
    (scba.py:647-658)."""
    md, mu, ml = m
    ne, n = md.shape[:2]
    cells = {}
    for side in ("left", "right"):
        xs = []
        for e in range(ne):
            if side == "left":
                cell = (md[e, 0], ml[e, 0], mu[e, 0])
            else:
                cell = (md[e, n - 1], mu[e, n - 2], ml[e, n - 2])
            x = _surface(cell, "W", side, e, surface_tol, cache, tol_memo)
            xs.append((cell, x))
        cells[side] = xs
    for side in ("left", "right"):
        j, o = (0, 1) if side == "left" else (n - 1, n - 2)
        for kind in ("<", ">"):
            bd, bu, bl = srcs[kind]
            for e in range(ne):
                (m_c, n_dn, n_up), x = cells[side][e]
                b_in = bl[e, 0] if side == "left" else bu[e, n - 2]      # B[o, j]
                b_out = bu[e, 0] if side == "left" else bl[e, n - 2]     # B[j, o]
                y = (n_dn @ x) @ b_in
                q0 = bd[e, j] - (y - _h(y))
                a = x @ n_dn
                q = (x @ q0) @ _h(x)
                if cache is None:
                    wl = stein_direct(a, q)
                else:
                    wl = memoized_obc(("W", side, e, kind), lambda: stein_direct(a, q),
                                      lambda w: q + (a @ w) @ _h(a), cache, cache.n_fpi(kind), tol_memo)
                t = n_dn @ x
                bd[e, j] = bd[e, j] + (-(t @ b_in) - (b_out @ _h(x)) @ _h(n_dn) + (n_dn @ wl) @ _h(n_dn))
    for side in ("left", "right"):
        j = 0 if side == "left" else n - 1
        for e in range(ne):
            (m_c, n_dn, n_up), x = cells[side][e]
            md[e, j] = md[e, j] - (n_dn @ x) @ n_up


# -- full SCBA iteration (scba.py:865-1216, sequential, memoizer off) ---------


def scba(h, v, energies, eta, mu_left, mu_right, kT, max_iter=1, tol=1e-12, mixing=0.3,
         surface_tol=1e-8, memoizer: tuple[int, int] | None = None, entry_cutoff: int | None = None):
    """scba_run(retarded_method='sancho', W surface by Sancho). ``memoizer``
    = (n_fpi_retarded, n_fpi_lg) enables the OBC memoizer with tol/10
    (scba.py:906-911); None = memoizer off. Returns the ScbaResult arrays (G
    at the start of the last iteration, mixed Sigma after it), 'residuals'
    and 'cache_stats_by_iteration'.

    ``entry_cutoff`` (NOT in the reference: the paper's r_cut nonzero set,
    PAPER.md:176, 207, the deviation ScbaOptions.entry_cutoff implements):
    G^<> and W^<> entries with |row - col| > entry_cutoff are zeroed after
    every gather, which makes P and Sigma vanish there too -- the same
    numbers as a computation on the restricted entry set."""
    energies = np.asarray(energies, dtype=float)
    ne = len(energies)
    de = (energies[-1] - energies[0]) / (ne - 1)
    n_b, bs = h[0].shape[0], h[0].shape[-1]
    rows, cols = entry_pattern(n_b, bs)
    diag_mask = rows == cols
    drop = np.abs(rows - cols) > entry_cutoff if entry_cutoff is not None else np.zeros(rows.shape, bool)
    trace_idx = [np.flatnonzero(diag_mask & (rows // bs == b)) for b in range(n_b)]
    n_ent = len(rows)
    sig = {k: np.zeros((n_ent, ne), complex) for k in ("lesser", "greater", "ret_upper", "ret_lower")}
    f_bath = fermi(energies, 0.5 * (mu_left + mu_right), kT)
    residuals = []
    cache = SurfaceCache(*memoizer) if memoizer is not None else None
    tol_memo = tol / 10.0
    stats_by_it = []
    for it in range(max_iter):
        sr = scatter_retarded(sig["ret_upper"], sig["ret_lower"], n_b, bs)
        sl = scatter_lg(sig["lesser"], n_b, bs)
        sg = scatter_lg(sig["greater"], n_b, bs)
        m, bl, bg = assemble_g(energies, eta, h, f_bath, sr=sr, sl=sl, sg=sg)
        obc = g_closure(m, bl, bg, energies, mu_left, mu_right, kT, surface_tol, cache, tol_memo)
        sol = rgf_selected(*m, {"<": bl, ">": bg}, symmetrize=True)
        result = {
            "g_r_diag": sol["xr_diag"], "g_r_upper": sol["xr_upper"], "g_r_lower": sol["xr_lower"],
            "g_lesser_diag": sol["x<_diag"], "g_lesser_upper": sol["x<_upper"],
            "g_greater_diag": sol["x>_diag"], "g_greater_upper": sol["x>_upper"],
            "sigma_obc_lesser_left": obc["left"][0], "sigma_obc_greater_left": obc["left"][1],
            "sigma_obc_lesser_right": obc["right"][0], "sigma_obc_greater_right": obc["right"][1],
        }
        gl = gather_entries(sol["x<_diag"], sol["x<_upper"])
        gg = gather_entries(sol["x>_diag"], sol["x>_upper"])
        gl[drop] = 0.0
        gg[drop] = 0.0
        pl, pg, pru, prl = polarization(gl, gg, diag_mask, de)
        pr = scatter_retarded(pru, prl, n_b, bs)
        mw, srcs = w_system(v, pr, scatter_lg(pl, n_b, bs), scatter_lg(pg, n_b, bs))
        w_closure(mw, srcs, surface_tol, cache, tol_memo)
        wsol = rgf_selected(*mw, srcs, symmetrize=True)
        wl = gather_entries(wsol["x<_diag"], wsol["x<_upper"])
        wg = gather_entries(wsol["x>_diag"], wsol["x>_upper"])
        wl[drop] = 0.0
        wg[drop] = 0.0
        raw = dict(zip(("lesser", "greater", "ret_upper", "ret_lower"), self_energy(gl, gg, wl, wg, diag_mask, de)))
        tr_old = {k: np.stack([sig[k][idx].sum(0) for idx in trace_idx]) for k in ("lesser", "greater")}
        for k in sig:
            sig[k] = (1.0 - mixing) * sig[k] + mixing * raw[k]
        tr_new = {k: np.stack([sig[k][idx].sum(0) for idx in trace_idx]) for k in ("lesser", "greater")}
        delta = max(float(np.max(np.abs(tr_new[k] - tr_old[k]))) for k in tr_new)
        scale = max(max(float(np.max(np.abs(tr_old[k]))) for k in tr_old),
                    max(float(np.max(np.abs(tr_new[k]))) for k in tr_new))
        residuals.append(delta / (scale + 1e-300))
        if cache is not None:
            stats_by_it.append(dict(cache.stats))
        if residuals[-1] < tol:
            break
    result.update({"sigma_" + k: v_ for k, v_ in sig.items()})
    result["residuals"] = np.asarray(residuals)
    result["cache_stats_by_iteration"] = stats_by_it
    return result
