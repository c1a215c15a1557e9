"""Test infrastructure: the sharded parareal decomposition restated on the numpy oracle.

Rank r owns slices [a_r, b_r).  Per iteration: fine/coarse stages for own slices, an
all-gather of the coarse payload (R(fine_next), coarse_next, flags), a replicated coarse
sweep that tracks R(next[n]) = R(fine_next[n]) + R(I(d_n)) instead of fine states, the
fine combine next[n] = fine_next[n] + I(d_n) on own slices and the boundary state sent to
rank r+1 — the algorithm of paratime_b200/csrc/driver.cu.  Used by the gloo CPU test to
check that the decomposition reproduces the reference's theta_engine (oracle)."""
from __future__ import annotations

import numpy as np
import torch.distributed as dist

from oracle import paratime_np as P


def partition(N, world, rank):
    chunk = -(-N // world)
    a = min(N + 1, 1 + rank * chunk)
    b = min(N + 1, a + chunk)
    return a, b


def _allgather(obj):
    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, obj)
    return out


def theta_sharded(init, sch: P.Schedule, t: P.Transfer, K, scheme, tol):
    rank, world = dist.get_rank(), dist.get_world_size()
    N = sch.n
    a, b = partition(N, world, rank)
    cc = sch.c_coarse
    RI = lambda s: (P.restrict_field(P.interpolate_field(s[0], t), t), P.restrict_field(P.interpolate_field(s[1], t), t))
    R = lambda s: (P.restrict_field(s[0], t), P.restrict_field(s[1], t))
    # iteration 0: coarse chain, replicated
    w0 = {}
    rn = R(init)
    for n in range(1, N + 1):
        try:
            w = P.propagate_coupling(rn[0], rn[1], cc, t.coarse, sch.dt_coarse, sch.m_coarse)
        except P.PropagationDiverged:
            w = P._nan_state(t.coarse)
        w0[n] = w
        rn = RI(w)
    cur = {0: init} if a == 1 else {}
    for n in range(a, b):
        cur[n] = P._interp_state(w0[n], t) if P.finite(*w0[n]) else P._nan_state(t.fine)
    # boundary: state a-1 from the previous rank
    cur = _shift(cur, a, b, init)
    corrector = P.empty_corrector()
    history = []
    for _ in range(K):
        fine_next, coarse_next = {}, {}
        for n in range(a, b):
            fine_next[n] = P.fine_stage(cur[n - 1], sch)
            coarse_next[n] = P.coarse_stage(cur[n - 1], sch, t)
        pay = {n: (R(fine_next[n]), coarse_next[n], P.finite(*fine_next[n]), P.finite(*coarse_next[n]))
               for n in range(a, b)}
        allpay = {}
        for d in _allgather(pay):
            allpay.update(d)
        keep = [n for n in range(1, N + 1) if allpay[n][2] and allpay[n][3]]
        if keep:
            F = np.stack([P.to_energy_components(*allpay[n][0], cc, t.coarse, scheme)[0] for n in keep], 1)
            G = np.stack([P.to_energy_components(*allpay[n][1], cc, t.coarse, scheme)[0] for n in keep], 1)
            corrector = P.update_svd(corrector, F, G, tol)
        applied = corrector
        d = {1: None}
        rn = allpay[1][0]
        for n in range(2, N + 1):
            try:
                w = P.propagate_coupling(rn[0], rn[1], cc, t.coarse, sch.dt_coarse, sch.m_coarse)
            except P.PropagationDiverged:
                w = P._nan_state(t.coarse)
            if not P.finite(*w) or not allpay[n][3] or not allpay[n][2]:
                d[n] = P._nan_state(t.coarse)
            else:
                cn = P._corrected_coarse_state(w, applied, cc, t.coarse, scheme, False)
                co = P._corrected_coarse_state(allpay[n][1], applied, cc, t.coarse, scheme, False)
                d[n] = (cn[0] - co[0], cn[1] - co[1])
            ri = RI(d[n])
            rn = (allpay[n][0][0] + ri[0], allpay[n][0][1] + ri[1])
        nxt = {0: init} if a == 1 else {}
        for n in range(a, b):
            if n == 1:
                nxt[n] = fine_next[1]
            else:
                i = P._interp_state(d[n], t)
                nxt[n] = (fine_next[n][0] + i[0], fine_next[n][1] + i[1])
            if not P.finite(*nxt[n]):
                nxt[n] = cur[n]
        nxt = _shift(nxt, a, b, init)
        history.append({n: nxt[n] for n in range(a, b)})
        cur = nxt
    return history


def _shift(states, a, b, init):
    """Send state b-1 to rank+1; receive state a-1 from rank-1 (object p2p over gloo)."""
    rank, world = dist.get_rank(), dist.get_world_size()
    objs = _allgather((b - 1, states.get(b - 1)) if b - 1 >= a else (None, None))
    if a > 1:
        for m, s in objs:
            if m == a - 1:
                states[a - 1] = s
    else:
        states[0] = init
    return states


def pml_plain_sharded(u0, v0, kf, m_f, kc, m_c, t, N, K):
    """The decomposition of csrc/pml.cu pml_parareal with slices block-sharded over the gloo ranks
    (numpy, test infrastructure): own fine and coarse stages, one all-gather of the coarse payload
    (C(R cur[n-1]) and R(fine_next[n])), the replicated coarse sweep, the own fine combine and the
    last own state sent to the next rank.  Returns {global n: state} of the own states per iteration."""
    import torch
    import torch.distributed as dist

    from oracle import paratime_np as P
    from oracle import pml_np as M

    rank, world = dist.get_rank(), dist.get_world_size()
    chunk = -(-N // world)
    a = min(N + 1, 1 + rank * chunk)
    b = min(N + 1, a + chunk)
    R = lambda s: tuple(P.restrict_field(f, t) for f in s)  # noqa: E731
    damped = (kf.zy[:, None] != 0.0) | (kf.zx[None, :] != 0.0)

    def I(s):  # noqa: E743  (px, py cut back to the layer, as oracle/pml_np.plain_parareal)
        u, v, px, py = (P.interpolate_field(f, t) for f in s)
        return u, v, np.where(damped, px, 0.0), np.where(damped, py, 0.0)

    Fp = lambda s: M.pml_steps(*s, kf, m_f)  # noqa: E731
    Cp = lambda s: M.pml_steps(*s, kc, m_c)  # noqa: E731
    z = np.zeros_like(u0)
    init = (u0, v0, z, z)
    cur, w = {}, R(init)
    if a == 1:
        cur[0] = init
    for n in range(1, b):
        w = Cp(w)
        if n >= a - 1:
            cur[n] = I(w)
    hist = []
    for _ in range(K):
        fine_next = {n: Fp(cur[n - 1]) for n in range(a, b)}
        payload = {n: (Cp(R(cur[n - 1])), R(fine_next[n])) for n in range(a, b)}
        gathered = [None] * world
        dist.all_gather_object(gathered, payload)
        allp = {}
        for g in gathered:
            allp.update(g)
        w, d = R(init), {}
        for n in range(1, N + 1):
            g = Cp(w)
            old, rf = allp[n]
            d[n] = tuple(x - y for x, y in zip(g, old))
            w = tuple(x + y for x, y in zip(rf, d[n]))
        nxt = {n: tuple(x + y for x, y in zip(fine_next[n], I(d[n]))) for n in range(a, b)}
        for n in range(a, b):  # non-finite iterates clamped to the previous one
            if not all(np.all(np.isfinite(f)) for f in nxt[n]):
                nxt[n] = cur[n]
        if a == 1:
            nxt[0] = init
        # boundary: the last own state to the next rank
        if rank + 1 < world and b <= N:
            dist.send(torch.from_numpy(np.stack(nxt[b - 1])), dst=rank + 1)
        if rank > 0 and a <= N:
            buf = torch.empty((4,) + u0.shape, dtype=torch.float64)
            dist.recv(buf, src=rank - 1)
            nxt[a - 1] = tuple(buf.numpy()[f].copy() for f in range(4))
        hist.append(nxt)
        cur = nxt
    return hist


# ---------------------------------------------------------------- row-sharded update_svd
# The decomposition of paratime_b200/csrc/procrustes.cu `update_svd_rows` restated on numpy: the
# tall matrices' rows are cut into SLABS fixed slabs of whole TSQR leaves, rank q owns the
# contiguous slabs [q SLABS/W, (q+1) SLABS/W).  Products over rows are per-slab partials gathered
# and summed in slab order; projections and rotations are row-local; each rank factors its own
# leaves, the stack of all leaves' R is gathered and reduced by every rank; the new factors' rows
# are gathered.  Everything small (H, its SVD, fix_signs) is replicated.

SLABS = 4


def _slab_tn(A_own, B_own, per):
    """A^T B over all rows: own slabs' partials -> all-gather -> summed in slab order."""
    slab = A_own.shape[0] // per
    parts = [A_own[s * slab:(s + 1) * slab].T @ B_own[s * slab:(s + 1) * slab] for s in range(per)]
    acc = None
    for ranks_parts in _allgather(parts):  # rank order == slab order (contiguous ownership)
        for p in ranks_parts:
            acc = p.copy() if acc is None else acc + p
    return acc


def _tsqr_rows(A_own, leaf_rows, drop_tol):
    """truncated_qr of the row-sharded block: own leaves, gathered R stack, own rows of Q."""
    n = A_own.shape[1]
    nbo = A_own.shape[0] // leaf_rows
    Ql, Rl = [], []
    for b in range(nbo):
        q, r = np.linalg.qr(A_own[b * leaf_rows:(b + 1) * leaf_rows])
        Ql.append(q)
        Rl.append(r)
    stacks = _allgather(np.vstack(Rl))
    S = np.vstack(stacks)
    Qs, R = P.truncated_qr(S, drop_tol)  # the pivoted decision is taken on the stack, replicated
    leaf0 = sum(s.shape[0] for s in stacks[:dist.get_rank()]) // n
    Q = np.vstack([Ql[b] @ Qs[(leaf0 + b) * n:(leaf0 + b + 1) * n] for b in range(nbo)])
    return Q, R


def update_svd_row_sharded(corr: P.Corrector, F, G, tol, leaf_rows):
    """procrustes.cpp:188-237 with the rows of U, V, F, G sharded over the ranks."""
    rank, world = dist.get_rank(), dist.get_world_size()
    rows = F.shape[0]
    assert rows % (SLABS * leaf_rows) == 0 and SLABS % world == 0
    per, own = SLABS // world, rows // world
    sl = slice(rank * own, (rank + 1) * own)
    U, V, Fo, Go = corr.X[sl], corr.Y[sl], F[sl], G[sl]
    r = corr.rank
    UF = _slab_tn(U, Fo, per)
    VG = _slab_tn(V, Go, per)
    fn = np.sqrt(sum(_allgather(float(np.sum(Fo * Fo)))))
    gn = np.sqrt(sum(_allgather(float(np.sum(Go * Go)))))
    QF, RF = _tsqr_rows(Fo - U @ UF, leaf_rows, 1e-14 * fn)
    QG, RG = _tsqr_rows(Go - V @ VG, leaf_rows, 1e-14 * gn)
    H = np.vstack([UF, RF]) @ np.vstack([VG, RG]).T
    H[np.arange(r), np.arange(r)] += corr.S
    Uh, sigma, Vh = P._thin_svd(H)
    keep = P._truncate(sigma, tol)
    Xo = np.hstack([U, QF]) @ Uh[:, :keep]
    Yo = np.hstack([V, QG]) @ Vh[:, :keep]
    X = np.vstack(_allgather(Xo))
    Y = np.vstack(_allgather(Yo))
    P.fix_signs(X, Y)
    return P.Corrector(X, sigma[:keep].copy(), Y, tol)
