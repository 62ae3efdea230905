"""Seeded synthetic KKT inputs for the condensed-KKT hot path (shared by tests, bench, smoke).

This module builds INPUTS only: sparsity patterns and values of W (Hessian of the
Lagrangian, lower triangle), J (constraint Jacobian), the barrier diagonals
Sigma_x = D_x = X^-1 U and Sigma_s = D_s = S^-1 V (eq K2), the
regularisations and right-hand sides.  It holds none of the method's arithmetic
(no condensation, no factorisation, no solve) -- both the oracle (oracle/) and the
CUDA path (paper_2405_14236_b200/) consume what it returns.

Workload recipes follow SURVEY.md §8(d) "Concrete synthetic inputs":

* C1  COPS bearing 50x50 (n=2500, bound-only m=0); W = 5-point FE stiffness with
      weight w_q = (1 + 0.1 cos xi1)^3 (COPS bearing, cited at P:123; formula is the
      generator's reading, reading R14).
* C2..C5  PGLIB-shaped polar ACOPF with the layout inferred from P:1359-1361
      (SURVEY.md §8 header): n = 2nb + 2ng + 4nl, m_e = 2nb + 4nl + 1, m_i = 3nl,
      nl = round(1.6056 nb), ng = round(0.08622 nb).
* Sigma magnitudes follow Prop. 1: active -> Theta(1/Xi), inactive -> Theta(Xi),
  Xi = 1e-8 (LiftedKKT) or Xi = 1/gamma (HyKKT, Assumption 2(b)).

Seed convention: seed = config_number * 1000 + instance.
"""
from __future__ import annotations

from dataclasses import dataclass, field
import numpy as np

__all__ = ["KKTInstance", "bearing", "acopf", "make_config", "tiny_random", "CONFIGS",
           "acopf_sizes", "redraw_values", "partition"]


@dataclass
class KKTInstance:
    name: str
    n: int
    m: int
    m_eq: int
    W_rowptr: np.ndarray          # int32 [n+1], lower-triangular CSR incl. full diagonal
    W_colind: np.ndarray          # int32 [nnzW], sorted within row, col <= row
    W_vals: np.ndarray            # float64 [nnzW] or [batch, nnzW]
    J_rowptr: np.ndarray          # int32 [m+1]
    J_colind: np.ndarray          # int32 [nnzJ], sorted within row
    J_vals: np.ndarray            # float64 [nnzJ] or [batch, nnzJ]
    Sigma_x: np.ndarray           # float64 [n] or [batch, n]
    Sigma_s: np.ndarray           # float64 [m - m_eq] or [batch, m - m_eq]
    delta_w: float = 0.0
    delta_c: float = 0.0
    gamma: float = 0.0
    b: np.ndarray | None = None       # condensed RHS [n] (or [batch, n])
    rbar1: np.ndarray | None = None   # HyKKT RHS block 1 [n]
    rbar2: np.ndarray | None = None   # HyKKT RHS block 2 [m_eq]
    batch: int = 1
    meta: dict = field(default_factory=dict)

    @property
    def nnzW(self) -> int:
        return int(self.W_rowptr[-1])

    @property
    def nnzJ(self) -> int:
        return int(self.J_rowptr[-1])

    def instance(self, k: int) -> "KKTInstance":
        """Instance k of a batch as a batch-1 KKTInstance (views)."""
        if self.batch == 1:
            return self
        pick = lambda a: None if a is None else a[k]
        return KKTInstance(f"{self.name}[{k}]", self.n, self.m, self.m_eq,
                           self.W_rowptr, self.W_colind, self.W_vals[k],
                           self.J_rowptr, self.J_colind, self.J_vals[k],
                           self.Sigma_x[k], self.Sigma_s[k], self.delta_w, self.delta_c,
                           self.gamma, pick(self.b), pick(self.rbar1), pick(self.rbar2),
                           1, dict(self.meta))


def _csr_from_coo(nrows, rows, cols, vals):
    """Sum duplicates, sort columns within rows; returns int32 rowptr/colind + float64 vals."""
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    vals = np.asarray(vals, dtype=np.float64)
    key = rows * (int(cols.max()) + 1 if cols.size else 1) + cols
    order = np.argsort(key, kind="stable")
    key, rows, cols, vals = key[order], rows[order], cols[order], vals[order]
    uniq, start = np.unique(key, return_index=True)
    sums = np.add.reduceat(vals, start) if vals.size else vals
    r = rows[start]
    c = cols[start]
    rowptr = np.zeros(nrows + 1, dtype=np.int64)
    np.add.at(rowptr, r + 1, 1)
    rowptr = np.cumsum(rowptr)
    return rowptr.astype(np.int32), c.astype(np.int32), sums


def _two_level(rng, size, active_mask, Xi):
    """Prop. 1 magnitudes: active -> U(0.5,2)/Xi, inactive -> U(0.5,2)*Xi."""
    u = rng.uniform(0.5, 2.0, size=size)
    return np.where(active_mask, u / Xi, u * Xi)


# --------------------------------------------------------------------------------------
# C1: COPS journal bearing
# --------------------------------------------------------------------------------------
def bearing(nx=50, ny=50, seed=1000, Xi=1e-8, band=(0.5, 0.8), ecc=0.1, b_len=10.0):
    """5-point FE stiffness of the COPS bearing (Dirichlet boundary, interior unknowns).

    Bound-only (m = 0): the condensed matrix is K = W + Sigma_x + delta_w I (P:415 with H empty).
    Sigma_x is U(0.5,2)/Xi on the cavitation band (variables at their bound) and U(0.5,2)*Xi
    elsewhere.
    """
    rng = np.random.default_rng(seed)
    n = nx * ny
    hx = 2 * np.pi / (nx + 1)
    hy = 2 * b_len / (ny + 1)
    wq = lambda xi1: (1.0 + ecc * np.cos(xi1)) ** 3
    idx = lambda i, j: j * nx + i          # i along xi1, j along xi2
    diag = np.zeros(n)
    rows, cols, vals = [], [], []
    I, Jg = np.meshgrid(np.arange(nx), np.arange(ny), indexing="ij")
    I = I.ravel(); Jg = Jg.ravel()
    p = idx(I, Jg)
    # horizontal edges (i-1/2 and i+1/2 midpoints), including edges to the boundary
    for di in (-1, +1):
        xm = (I + 1 + 0.5 * di) * hx
        c = wq(xm) * hy / hx
        np.add.at(diag, p, c)
        inside = (I + di >= 0) & (I + di < nx)
        q = idx(I + di, Jg)
        sel = inside & (q < p)
        rows.append(p[sel]); cols.append(q[sel]); vals.append(-c[sel])
    for dj in (-1, +1):
        xm = (I + 1) * hx
        c = wq(xm) * hx / hy
        np.add.at(diag, p, c)
        inside = (Jg + dj >= 0) & (Jg + dj < ny)
        q = idx(I, Jg + dj)
        sel = inside & (q < p)
        rows.append(p[sel]); cols.append(q[sel]); vals.append(-c[sel])
    rows.append(np.arange(n)); cols.append(np.arange(n)); vals.append(diag)
    Wp, Wc, Wv = _csr_from_coo(n, np.concatenate(rows), np.concatenate(cols), np.concatenate(vals))
    frac = (I / nx)
    active = (frac >= band[0]) & (frac < band[1])

    def draw(rng):
        Sx = np.empty(n)
        Sx[p] = _two_level(rng, n, active, Xi)
        return np.zeros(0), Wv, Sx, np.zeros(0), rng.standard_normal(n), None, None

    _, _, Sx, _, b, _, _ = draw(rng)
    Jp = np.zeros(1, dtype=np.int32)
    inst = KKTInstance("C1-bearing-%dx%d" % (nx, ny), n, 0, 0, Wp, Wc, Wv, Jp,
                       np.zeros(0, np.int32), np.zeros(0), Sx, np.zeros(0), b=b,
                       meta=dict(kind="bearing", nx=nx, ny=ny, Xi=Xi, seed=seed, band=band))
    inst.meta["_draw"] = draw
    return inst


# --------------------------------------------------------------------------------------
# COPS elec (NEXT-3): the dense instance
# --------------------------------------------------------------------------------------
def elec(npts=400, seed=7000, Xi=1e-8):
    """Synthetic COPS elec shape (np electrons on the unit sphere: n = 3 np,
    m = np): the Hessian of the Coulomb energy couples every pair of points, so W (and K) is
    fully dense ("some are fully dense (elec)").  LiftedKKT form (m_eq = 0): row i
    of J is the gradient 2 p_i of the sphere constraint of point i (3 entries), relaxed and
    active (D = U(0.5,2)/Xi).  The points have no bounds, so Sigma_x is tiny
    (U(0.5,2)*Xi).  W = A A^T / n + diag(row |.| sum + 1) with A ~ N(0,1) (SPD, R17)."""
    rng = np.random.default_rng(seed)
    n, m = 3 * npts, npts
    A = rng.standard_normal((n, n)) / np.sqrt(n)
    Wd = A @ A.T
    Wd += np.diag(np.abs(Wd).sum(1) + 1.0)
    ii, jj = np.tril_indices(n)
    Wp, Wc, Wv = _csr_from_coo(n, ii, jj, Wd[ii, jj])
    pts = rng.standard_normal((npts, 3))
    pts /= np.linalg.norm(pts, axis=1, keepdims=True)
    Jp = (np.arange(m + 1) * 3).astype(np.int32)
    Jc = (3 * np.repeat(np.arange(m), 3) + np.tile(np.arange(3), m)).astype(np.int32)

    def draw(rng):
        P = rng.standard_normal((npts, 3))
        P /= np.linalg.norm(P, axis=1, keepdims=True)
        Jv = (2.0 * P).ravel()
        Sx = rng.uniform(0.5, 2.0, n) * Xi
        Ss = rng.uniform(0.5, 2.0, m) / Xi
        return Jv, Wv, Sx, Ss, rng.standard_normal(n), None, None

    Jv, _, Sx, Ss, b, _, _ = draw(rng)
    inst = KKTInstance("elec-%d" % npts, n, m, 0, Wp, Wc, Wv, Jp, Jc, Jv, Sx, Ss, b=b,
                       meta=dict(kind="elec", npts=npts, Xi=Xi, seed=seed))
    inst.meta["_draw"] = draw
    return inst


# --------------------------------------------------------------------------------------
# ACOPF-shaped (C2..C5)
# --------------------------------------------------------------------------------------
def acopf_sizes(nb):
    nl = int(round(1.6056 * nb))
    ng = max(1, int(round(0.08622 * nb)))
    n = 2 * nb + 2 * ng + 4 * nl
    m_e = 2 * nb + 4 * nl + 1
    m_i = 3 * nl
    return dict(nb=nb, nl=nl, ng=ng, n=n, m_e=m_e, m_i=m_i, m=m_e + m_i)


def _network(nb, nl, ng, rng):
    """Jittered sqrt(nb) x sqrt(nb) grid; random spanning tree + extra 4/8-neighbour edges."""
    side = int(np.ceil(np.sqrt(nb)))
    k = np.arange(nb)
    x, y = k % side, k // side
    cand = []
    for dx, dy, kind in ((1, 0, 4), (0, 1, 4), (1, 1, 8), (-1, 1, 8)):
        x2, y2 = x + dx, y + dy
        ok = (x2 >= 0) & (x2 < side)
        k2 = y2 * side + x2
        ok &= (k2 < nb)
        cand.append(np.stack([k[ok], k2[ok], np.full(ok.sum(), kind)], axis=1))
    cand = np.concatenate(cand)
    four = cand[cand[:, 2] == 4]
    # Kruskal over random weights on the 4-neighbour edges -> random spanning tree
    order = rng.permutation(len(four))
    parent = np.arange(nb)

    def find(a):
        while parent[a] != a:
            parent[a] = parent[parent[a]]
            a = parent[a]
        return a
    tree = []
    for e in order:
        a, b = four[e, 0], four[e, 1]
        ra, rb = find(a), find(b)
        if ra != rb:
            parent[ra] = rb
            tree.append(e)
            if len(tree) == nb - 1:
                break
    assert len(tree) == nb - 1, "grid not connected"
    in_tree = np.zeros(len(four), bool)
    in_tree[tree] = True
    rest = np.concatenate([four[~in_tree], cand[cand[:, 2] == 8]])
    extra = rest[rng.choice(len(rest), size=nl - (nb - 1), replace=False)]
    edges = np.concatenate([four[in_tree][:, :2], extra[:, :2]])
    flip = rng.random(len(edges)) < 0.5
    fr = np.where(flip, edges[:, 1], edges[:, 0])
    to = np.where(flip, edges[:, 0], edges[:, 1])
    perm = rng.permutation(len(edges))        # branch numbering is random
    fr, to = fr[perm], to[perm]
    gens = np.sort(rng.choice(nb, size=ng, replace=False))
    return fr.astype(np.int64), to.astype(np.int64), gens.astype(np.int64)


def acopf(nb, seed, hykkt=False, gamma=1e7, Xi=None, relaxed_active=1.0,
          ineq_active=None, x_active=None, delta_w=0.0, delta_c=0.0, batch=1,
          name=None, _pattern_rng_seed=None):
    """Synthetic polar-ACOPF condensed-KKT inputs.

    Variables:  va[nb] vm[nb] pg[ng] qg[ng] pft[nl] qft[nl] ptf[nl] qtf[nl]
    Rows (equalities first):  ref-angle (1), P balance (nb), Q balance (nb),
                              flow definitions (4 nl)            -> m_e = 2nb + 4nl + 1
                              thermal from/to (2 nl), angle difference (nl)   -> m_i = 3 nl
    LiftedKKT (hykkt=False): every row is an inequality (m_eq = 0); the m_e relaxed equalities
      -tau <= g <= tau become one row each with combined weight (reading R2).
    HyKKT (hykkt=True):   rows [0, m_e) are the equalities G weighted by gamma (m_eq = m_e).
    """
    s = acopf_sizes(nb)
    nl, ng, n, m_e, m_i = s["nl"], s["ng"], s["n"], s["m_e"], s["m_i"]
    prng = np.random.default_rng(seed if _pattern_rng_seed is None else _pattern_rng_seed)
    fr, to, gens = _network(nb, nl, ng, prng)
    VA, VM, PG, QG = 0, nb, 2 * nb, 2 * nb + ng
    PFT, QFT, PTF, QTF = 2 * nb + 2 * ng, 2 * nb + 2 * ng + nl, 2 * nb + 2 * ng + 2 * nl, 2 * nb + 2 * ng + 3 * nl
    L = np.arange(nl)

    # ---- Jacobian pattern (row, col, kind) ----
    # kind codes pick the value distribution (SURVEY.md §8(d) C2 "Jacobian values")
    r_list, c_list, k_list = [], [], []
    def add(r, c, kind):
        r_list.append(np.asarray(r, np.int64)); c_list.append(np.asarray(c, np.int64))
        k_list.append(np.full(np.size(r), kind, np.int8))
    row = 0
    add([0], [VA + 0], 3)                           # reference angle row: va_ref
    row = 1
    PB, QB = row, row + nb
    # balance rows: +1 generator, -1 flow, vm ~ N(0, 0.1^2)
    add(PB + np.arange(nb), VM + np.arange(nb), 1)
    add(QB + np.arange(nb), VM + np.arange(nb), 1)
    add(PB + gens, PG + np.arange(ng), 0)
    add(QB + gens, QG + np.arange(ng), 0)
    add(PB + fr, PFT + L, 2); add(PB + to, PTF + L, 2)
    add(QB + fr, QFT + L, 2); add(QB + to, QTF + L, 2)
    row = 1 + 2 * nb
    for blk, var in enumerate((PFT, QFT, PTF, QTF)):
        rr = row + blk * nl + L
        add(rr, var + L, 2)                          # -1 on the flow variable
        for vv in (VM + fr, VM + to, VA + fr, VA + to):
            add(rr, vv, 4)                           # voltages ~ N(0, 10^2)
    row = m_e
    add(row + L, PFT + L, 5); add(row + L, QFT + L, 5)          # thermal from
    add(row + nl + L, PTF + L, 5); add(row + nl + L, QTF + L, 5)  # thermal to
    add(row + 2 * nl + L, VA + fr, 3); add(row + 2 * nl + L, VA + to, 6)  # angle diff +1/-1
    m = m_e + m_i
    R = np.concatenate(r_list); C = np.concatenate(c_list); Kd = np.concatenate(k_list)
    order = np.lexsort((C, R))
    R, C, Kd = R[order], C[order], Kd[order]
    # (no duplicates by construction: one gen per bus, one flow var per branch end)
    keyd = R * n + C
    assert np.all(np.diff(keyd) > 0), "duplicate Jacobian entries"
    Jp = np.zeros(m + 1, np.int64); np.add.at(Jp, R + 1, 1); Jp = np.cumsum(Jp).astype(np.int32)
    Jc = C.astype(np.int32)

    # ---- W pattern: full diagonal + per-branch 4x4 block over (vm_f, vm_t, va_f, va_t) ----
    blk = np.stack([VM + fr, VM + to, VA + fr, VA + to], axis=1)
    wr, wc = [], []
    for a in range(4):
        for b in range(a):
            i, j = blk[:, a], blk[:, b]
            wr.append(np.maximum(i, j)); wc.append(np.minimum(i, j))
    wr = np.concatenate(wr); wc = np.concatenate(wc)
    offkey = np.unique(wr * n + wc)
    off_r, off_c = offkey // n, offkey % n
    Wr = np.concatenate([off_r, np.arange(n)]); Wc = np.concatenate([off_c, np.arange(n)])
    o = np.lexsort((Wc, Wr)); Wr, Wc = Wr[o], Wc[o]
    Wp = np.zeros(n + 1, np.int64); np.add.at(Wp, Wr + 1, 1); Wp = np.cumsum(Wp).astype(np.int32)
    Wcol = Wc.astype(np.int32)
    is_diag = (Wr == Wc)

    m_eq = m_e if hykkt else 0
    if Xi is None:
        Xi = (1.0 / gamma) if hykkt else 1e-8
    if ineq_active is None:
        ineq_active = 0.005 if hykkt else 0.10
    if x_active is None:                 # HyKKT: one active fraction for bounds and inequalities
        x_active = ineq_active if hykkt else 0.05

    def draw(rng):
        # J values by kind
        v = np.empty(len(Kd))
        z = lambda k: Kd == k
        v[z(0)] = 1.0
        v[z(1)] = rng.normal(0.0, 0.1, z(1).sum())
        v[z(2)] = -1.0
        v[z(3)] = 1.0
        v[z(4)] = rng.normal(0.0, 10.0, z(4).sum())
        v[z(5)] = rng.normal(0.0, 1.0, z(5).sum())
        v[z(6)] = -1.0
        # W: off-diagonal N(0,1); diagonal = row-abs-sum (both triangles) + 1  => lambda_min >= 1
        wv = np.zeros(len(Wr))
        offm = ~is_diag
        wv[offm] = rng.normal(0.0, 1.0, offm.sum())
        rs = np.zeros(n)
        np.add.at(rs, Wr[offm], np.abs(wv[offm])); np.add.at(rs, Wc[offm], np.abs(wv[offm]))
        wv[is_diag] = rs[Wr[is_diag]] + 1.0
        Sx = _two_level(rng, n, rng.random(n) < x_active, Xi)
        if hykkt:
            Ss = _two_level(rng, m_i, rng.random(m_i) < ineq_active, Xi)
        else:
            act = np.concatenate([rng.random(m_e) < relaxed_active, rng.random(m_i) < ineq_active])
            Ss = _two_level(rng, m, act, Xi)
        b = rng.standard_normal(n)
        r1 = rng.standard_normal(n)
        r2 = rng.standard_normal(m_eq)
        return v, wv, Sx, Ss, b, r1, r2

    family = batch > 1 or _pattern_rng_seed is not None   # batch family: instance k <- seed + k
    outs = [draw(np.random.default_rng(seed + k if family else seed + 7919)) for k in range(batch)]
    stack = (lambda i: outs[0][i]) if batch == 1 else (lambda i: np.stack([o[i] for o in outs]))
    inst = KKTInstance(name or ("acopf-%d%s" % (nb, "-hykkt" if hykkt else "")), n, m, m_eq,
                       Wp, Wcol, stack(1), Jp, Jc, stack(0), stack(2), stack(3),
                       delta_w, delta_c, gamma if hykkt else 0.0, stack(4),
                       stack(5) if hykkt else None, stack(6) if hykkt else None, batch,
                       meta=dict(kind="acopf", seed=seed, Xi=Xi, relaxed_active=relaxed_active,
                                 ineq_active=ineq_active, x_active=x_active, hykkt=hykkt, **s))
    inst.meta["_draw"] = draw
    return inst


def redraw_values(inst: KKTInstance, seed: int) -> KKTInstance:
    """New values on the same pattern ("successive IPM iterations")."""
    draw = inst.meta.get("_draw")
    if draw is None:
        raise ValueError("instance has no value generator")
    v, wv, Sx, Ss, b, r1, r2 = draw(np.random.default_rng(seed))
    out = KKTInstance(inst.name, inst.n, inst.m, inst.m_eq, inst.W_rowptr, inst.W_colind, wv,
                      inst.J_rowptr, inst.J_colind, v, Sx, Ss, inst.delta_w, inst.delta_c,
                      inst.gamma, b, r1 if inst.m_eq else None, r2 if inst.m_eq else None, 1,
                      dict(inst.meta))
    return out


def tiny_random(n, m, m_eq=0, density=0.3, seed=0, Xi=1e-4, hykkt_gamma=0.0,
                delta_w=0.0, delta_c=0.0, w_psd=True):
    """Tiny random instance (n <= ~50) for brute-force pins. W SPD by diagonal dominance."""
    rng = np.random.default_rng(seed)
    A = (rng.random((n, n)) < density)
    A = np.tril(A | A.T, -1)
    ri, ci = np.nonzero(A)
    off = rng.normal(0.0, 1.0, len(ri))
    rs = np.zeros(n); np.add.at(rs, ri, np.abs(off)); np.add.at(rs, ci, np.abs(off))
    dg = rs + 1.0 if w_psd else rng.normal(0.0, 1.0, n)
    Wp, Wc, Wv = _csr_from_coo(n, np.concatenate([ri, np.arange(n)]),
                               np.concatenate([ci, np.arange(n)]), np.concatenate([off, dg]))
    rows, cols = [], []
    for r in range(m):
        k = max(1, rng.binomial(n, min(1.0, 3.0 / max(n, 1))))
        c = np.sort(rng.choice(n, size=min(k, n), replace=False))
        rows.append(np.full(len(c), r)); cols.append(c)
    if m:
        Jp, Jc, Jv = _csr_from_coo(m, np.concatenate(rows), np.concatenate(cols),
                                   rng.normal(0.0, 1.0, sum(len(c) for c in cols)))
    else:
        Jp, Jc, Jv = np.zeros(1, np.int32), np.zeros(0, np.int32), np.zeros(0)
    Sx = _two_level(rng, n, rng.random(n) < 0.3, Xi)
    Ss = _two_level(rng, m - m_eq, rng.random(m - m_eq) < 0.5, Xi)
    return KKTInstance("tiny-%d-%d-%d" % (n, m, seed), n, m, m_eq, Wp, Wc, Wv, Jp, Jc, Jv, Sx, Ss,
                       delta_w, delta_c, hykkt_gamma, rng.standard_normal(n),
                       rng.standard_normal(n) if m_eq else None,
                       rng.standard_normal(m_eq) if m_eq else None,
                       meta=dict(kind="tiny", seed=seed))


CONFIGS = {
    "C1": "COPS bearing 50x50, LiftedKKT/direct, bound-only (n=2500)",
    "C2": "ACOPF ~2,000 buses, LiftedKKT",
    "C2s": "ACOPF ~2,000 buses, LiftedKKT, stress (50% relaxed rows active)",
    "C3": "ACOPF ~10,000 buses, HyKKT (gamma=1e4..1e7)",
    "C4": "ACOPF ~78,484 buses, LiftedKKT",
    "C5": "batch of 512 x ACOPF 500 buses (same pattern)",
    "C6": "NEXT-3: COPS bearing 800x800 (n=640,000, bound-only)",
    "C7": "NEXT-3: COPS elec 800 points, dense (n=2,400, m=800), LiftedKKT",
}


def partition(total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous block partition of `total` batch instances over `world` ranks:
    rank k gets [k*total//world, (k+1)*total//world)."""
    return rank * total // world, (rank + 1) * total // world


def make_config(name: str, instance: int = 0, gamma: float = 1e7, batch: int | None = None,
                **kw) -> KKTInstance:
    """Build configuration C1..C5; seed = config_number*1000 + instance."""
    num = int(name[1])
    seed = num * 1000 + instance
    if name == "C1":
        return bearing(50, 50, seed=seed, **kw)
    if name == "C2":
        return acopf(2000, seed, name="C2-acopf2000", **kw)
    if name == "C2s":
        return acopf(2000, seed, relaxed_active=0.5, name="C2s-acopf2000-stress", **kw)
    if name == "C3":
        return acopf(10000, seed, hykkt=True, gamma=gamma, name="C3-acopf10000-hykkt", **kw)
    if name == "C4":
        return acopf(78484, seed, name="C4-acopf78484", **kw)
    if name == "C5":
        # instance k of the batch draws its values from seed 5000 + instance + k, so any block of
        # a partition reproduces the same instances as the full batch (bitwise)
        return acopf(500, seed, batch=512 if batch is None else batch, name="C5-acopf500-batch",
                     _pattern_rng_seed=5000, **kw)
    if name == "C6":
        return bearing(800, 800, seed=seed, **kw)
    if name == "C7":
        return elec(800, seed=seed, **kw)
    raise KeyError(name)
