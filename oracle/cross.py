"""Greedy restricted TT-cross, restated (TEST INFRASTRUCTURE ONLY).

Follows ``ttpmf.tt_algorithms.greedy_cross`` (tt_algorithms.py:463-596) and
its helpers decision for decision and draw for draw, using numpy's own
``Generator`` so that a run is bit-replayable against the reference.
Constants: tt_algorithms.py:49-58.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import scipy.linalg

from oracle.ttcore import at_indices

N_INIT = 32        # _INIT_PROBES
N_CAND = 10        # _CAND_SET
ROOK = 2           # _ROOK_ITERS
SCAN = 1024        # _SCAN_CAP
BATCH = 24         # _BATCH_MAX
INJECT = 8         # _INJECT_MAX
FRESH = 128        # _SWEEP_FRESH
SAMPLE = 4096      # _SWEEP_SAMPLE
GATE = 32768       # _GATE_SAMPLE
TINY = np.finfo(float).tiny


@dataclass
class CrossOut:
    cores: list
    achieved_error: float
    evaluator_calls: int
    sweeps: int
    converged: bool


class Memo:
    """Memoised counted evaluator.  tt_algorithms.py:137-208.

    Keys are the C-order flat index: int64 via ravel_multi_index (as the
    reference computes them) when the grid has fewer than 2**63 cells, exact
    Python ints otherwise (the reference overflows there, F6).  Misses of a
    call are deduplicated, sorted ascending and appended in that order --
    the insertion order is what ``sample`` draws positions from.
    """

    def __init__(self, shape, fn):
        self.shape = tuple(int(n) for n in shape)
        self.fn = fn
        self.slot: dict[int, int] = {}
        self.keys: list[int] = []
        self.vals = np.empty(1024)
        self.calls = 0
        self.max_abs = 0.0
        self.small = math.prod(self.shape) < 2 ** 63
        w = [1] * len(self.shape)
        for k in range(len(self.shape) - 2, -1, -1):
            w[k] = w[k + 1] * self.shape[k + 1]
        self.weights = w

    def flat(self, idx):
        if self.small:
            return np.ravel_multi_index(tuple(np.asarray(idx, dtype=np.intp).T), self.shape)
        return [sum(int(i) * w for i, w in zip(row, self.weights)) for row in idx.tolist()]

    def unflat(self, keys) -> np.ndarray:
        if self.small:
            keys = np.asarray(keys, dtype=np.int64)
            if keys.size == 0:
                return np.empty((0, len(self.shape)), dtype=np.intp)
            return np.column_stack(np.unravel_index(keys, self.shape)).astype(np.intp)
        out = np.empty((len(keys), len(self.shape)), dtype=np.intp)
        for j, key in enumerate(keys):
            for k, w in enumerate(self.weights):
                out[j, k], key = divmod(key, w)
        return out

    def __call__(self, idx) -> np.ndarray:
        idx = np.asarray(idx, dtype=np.intp).reshape(-1, len(self.shape))
        flat = self.flat(idx)
        keys = flat.tolist() if self.small else flat
        get = self.slot.get
        if self.small:
            pos = np.fromiter((get(k, -1) for k in keys), dtype=np.int64, count=len(keys))
            miss = np.unique(flat[pos < 0]).tolist() if (pos < 0).any() else []
        else:
            miss = sorted({k for k in keys if k not in self.slot})
        if miss:
            v = np.asarray(self.fn(self.unflat(miss)), dtype=float).reshape(-1)
            if v.shape != (len(miss),):
                raise ValueError("evaluator returned wrong number of values")
            if not np.all(np.isfinite(v)):
                raise ValueError("evaluator returned a non-finite value")
            self.calls += len(miss)
            self.max_abs = max(self.max_abs, float(np.max(np.abs(v))))
            base = len(self.keys)
            if base + len(miss) > len(self.vals):
                grown = np.empty(max(base + len(miss), 2 * len(self.vals)))
                grown[:base] = self.vals[:base]
                self.vals = grown
            self.vals[base:base + len(miss)] = v
            self.slot.update(zip(miss, range(base, base + len(miss))))
            self.keys.extend(miss)
            if self.small:
                pos = np.fromiter((get(k) for k in keys), dtype=np.int64, count=len(keys))
        if not self.small:
            pos = np.array([self.slot[k] for k in keys], dtype=np.int64)
        return self.vals[pos]

    def sample(self, rng, count):
        n = len(self.keys)
        sel = rng.choice(n, size=count, replace=False) if n > count else np.arange(n)
        return self.unflat([self.keys[j] for j in sel]), self.vals[sel].copy()


def _cartesian(left, n, right) -> np.ndarray:
    """(A*n*C, a+1+c) indices, suffix fastest.  tt_algorithms.py:211-224."""
    a, la = left.shape
    c, lc = right.shape
    out = np.empty((a, n, c, la + 1 + lc), dtype=np.intp)
    out[..., :la] = left[:, None, None, :]
    out[..., la] = np.arange(n)[None, :, None]
    out[..., la + 1:] = right[None, None, :, :]
    return out.reshape(-1, la + 1 + lc)


def _arr(tuples, width) -> np.ndarray:
    return np.array(tuples, dtype=np.intp).reshape(len(tuples), width)


class Skeleton:
    """Nested pivot sets, fibres, pivot blocks and cores.  tt_algorithms.py:232-338."""

    def __init__(self, memo: Memo, pivot):
        self.m = memo
        self.n = memo.shape
        d = len(self.n)
        self.d = d
        self.I = [None] + [[tuple(pivot[:b])] for b in range(1, d)]   # row prefixes per bond
        self.J = [None] + [[tuple(pivot[b:])] for b in range(1, d)]   # column suffixes per bond
        self.fib = [memo(_cartesian(self.lhs(k), self.n[k], self.rhs(k))).reshape(
            len(self.left(k)), self.n[k], len(self.right(k))) for k in range(d)]
        self.piv = [None] + [self.block(self.I[b], self.J[b]) for b in range(1, d)]
        self.core = [None] * d
        for k in range(d):
            self.solve(k)

    def left(self, k):
        return [()] if k == 0 else self.I[k]

    def right(self, k):
        return [()] if k == self.d - 1 else self.J[k + 1]

    def lhs(self, k):
        return _arr(self.left(k), k)

    def rhs(self, k):
        return _arr(self.right(k), self.d - k - 1)

    def rank(self, b):
        return len(self.I[b])

    def limit(self, b, max_rank):
        return min(max_rank, len(self.left(b - 1)) * self.n[b - 1],
                   self.n[b] * len(self.right(b)))

    def block(self, rows, cols):
        b = len(rows[0])
        blk = np.empty((len(rows), len(cols), self.d), dtype=np.intp)
        blk[..., :b] = _arr(rows, b)[:, None, :]
        blk[..., b:] = _arr(cols, self.d - b)[None, :, :]
        return self.m(blk.reshape(-1, self.d)).reshape(len(rows), len(cols))

    def solve(self, k):
        f = self.fib[k]
        if k == self.d - 1:
            self.core[k] = f
            return
        r = f.shape[2]
        g = scipy.linalg.lstsq(self.piv[k + 1].T, f.reshape(-1, r).T,
                               lapack_driver="gelsy")[0].T
        self.core[k] = g.reshape(f.shape[0], self.n[k], r)

    def grow(self, b, rows, cols):
        oi, oj = self.I[b], self.J[b]
        rb = self.block(rows, oj)
        cb = self.block(oi + rows, cols)
        self.piv[b] = np.concatenate([
            np.concatenate([self.piv[b], cb[:len(oi)]], axis=1),
            np.concatenate([rb, cb[len(oi):]], axis=1)], axis=0)
        self.I[b] = oi + rows
        self.J[b] = oj + cols
        rhs = self.rhs(b)
        slab = self.m(_cartesian(_arr(rows, b), self.n[b], rhs))
        self.fib[b] = np.concatenate(
            [self.fib[b], slab.reshape(len(rows), self.n[b], len(rhs))], axis=0)
        lhs = self.lhs(b - 1)
        slab = self.m(_cartesian(lhs, self.n[b - 1], _arr(cols, self.d - b)))
        self.fib[b - 1] = np.concatenate(
            [self.fib[b - 1], slab.reshape(len(lhs), self.n[b - 1], len(cols))], axis=2)
        self.solve(b - 1)
        self.solve(b)

    def cores(self):
        return list(self.core)


def _hunt(sk: Skeleton, b: int, rng):
    """Random 10x10 candidate block + rook refinement.  tt_algorithms.py:341-421."""
    d = sk.d
    pre = sk.lhs(b - 1)
    suf = sk.rhs(b)
    nl, nr = sk.n[b - 1], sk.n[b]
    nrow = len(pre) * nl
    ncol = nr * len(suf)
    ns = len(suf)
    gl = sk.core[b - 1].reshape(nrow, -1)
    fr = sk.fib[b].reshape(-1, ncol)

    def cells(rf, cf):
        idx = np.empty((len(rf), d), dtype=np.intp)
        idx[:, :b - 1] = pre[rf // nl]
        idx[:, b - 1] = rf % nl
        idx[:, b] = cf // ns
        idx[:, b + 1:] = suf[cf % ns]
        return idx

    def err(rf, cf):
        approx = np.einsum("ir,ri->i", gl[rf], fr[:, cf])
        return np.abs(sk.m(cells(rf, cf)) - approx)

    qr_, qc = min(N_CAND, nrow), min(N_CAND, ncol)
    cr = rng.choice(nrow, size=qr_, replace=False)
    cc = rng.choice(ncol, size=qc, replace=False)
    br = np.repeat(cr, qc)
    bc = np.tile(cc, qr_)
    e = err(br, bc)
    order = np.argsort(e)[::-1]
    cand = [(int(br[i]), int(bc[i]), float(e[i])) for i in order]
    seen = cand[0][2] if cand else 0.0
    rb, cb = (cand[0][0], cand[0][1]) if cand else (0, 0)
    for _ in range(ROOK):
        rows = rng.choice(nrow, size=SCAN, replace=False) if nrow > SCAN else np.arange(nrow)
        ec = err(rows, np.full(len(rows), cb))
        rn = int(rows[int(np.argmax(ec))])
        cols = rng.choice(ncol, size=SCAN, replace=False) if ncol > SCAN else np.arange(ncol)
        er = err(np.full(len(cols), rn), cols)
        cn = int(cols[int(np.argmax(er))])
        seen = max(seen, max(float(np.max(ec)), float(np.max(er))))
        if rn == rb and cn == cb:
            break
        rb, cb = rn, cn
    cand.insert(0, (rb, cb, float(err(np.array([rb]), np.array([cb]))[0])))

    def split(rf, cf):
        return (tuple(pre[rf // nl]) + (rf % nl,), (cf // ns,) + tuple(suf[cf % ns]))

    return cand, seen, split


def _check(sk: Skeleton, cores, rng, count, top=1):
    """Worst errors on a random cache subsample.  tt_algorithms.py:424-433."""
    idx, vals = sk.m.sample(rng, count)
    e = np.abs(vals - at_indices(cores, idx))
    order = np.argsort(e)[::-1][:top]
    return [(float(e[j]), tuple(int(i) for i in idx[j])) for j in order]


def _inject(sk: Skeleton, offenders, thr, max_rank) -> bool:
    """Adopt wrong cached cells as pivots.  tt_algorithms.py:436-460."""
    pend: dict[int, tuple[list, list]] = {}
    for e, cell in offenders:
        if e <= thr:
            break
        for b in range(1, sk.d):
            pr, pc = pend.setdefault(b, ([], []))
            if sk.rank(b) + len(pr) >= sk.limit(b, max_rank):
                continue
            row, col = cell[:b], cell[b:]
            if row in sk.I[b] or row in pr or col in sk.J[b] or col in pc:
                continue
            pr.append(row)
            pc.append(col)
            break
    grew = False
    for b in sorted(pend):
        if pend[b][0]:
            sk.grow(b, *pend[b])
            grew = True
    return grew


def greedy_cross(shape, fn, tol=1e-6, max_rank=40, max_sweeps=60, rng_seed=0,
                 validation_count=100, seed_indices=None) -> CrossOut:
    """tt_algorithms.py:463-596 (argument names follow CrossConfig)."""
    shape = tuple(int(n) for n in shape)
    d = len(shape)
    memo = Memo(shape, fn)
    rng = np.random.default_rng(rng_seed)
    if d == 1:
        v = memo(np.arange(shape[0], dtype=np.intp)[:, None])
        return CrossOut([v.reshape(1, -1, 1)], 0.0, memo.calls, 0, True)
    probes = rng.integers(0, shape, size=(N_INIT + 4 * d, d))
    if seed_indices is not None:
        probes = np.concatenate([probes, np.asarray(seed_indices, dtype=np.intp).reshape(-1, d)])
    v = memo(probes)
    sk = Skeleton(memo, tuple(int(i) for i in probes[int(np.argmax(np.abs(v)))]))
    fresh = int(min(FRESH, max(4 * d, math.prod(shape) // 64)))

    sweeps, converged, clean = 0, False, 0
    best_err, best = math.inf, None
    for _ in range(max_sweeps):
        sweeps += 1
        swe = 0.0
        grew = False
        full = True
        for b in range(1, d):
            r = sk.rank(b)
            lim = sk.limit(b, max_rank)
            if r >= lim:
                continue
            full = False
            cand, seen, split = _hunt(sk, b, rng)
            swe = max(swe, seen)
            thr = tol * max(memo.max_abs, TINY)
            cap = min(BATCH, max(1, r // 2), lim - r)
            nr_, nc_ = [], []
            for rf, cf, e in cand:
                if e <= thr or len(nr_) >= cap:
                    break
                row, col = split(rf, cf)
                if row in sk.I[b] or row in nr_ or col in sk.J[b] or col in nc_:
                    continue
                nr_.append(row)
                nc_.append(col)
            if nr_:
                sk.grow(b, nr_, nc_)
                grew = True
        memo(rng.integers(0, shape, size=(fresh, d)))
        thr = tol * max(memo.max_abs, TINY)
        now = sk.cores()
        off = _check(sk, now, rng, SAMPLE, top=INJECT)
        swe = max(swe, off[0][0])
        if swe < best_err:
            best_err, best = swe, now
        if off[0][0] > thr:
            grew = _inject(sk, off, thr, max_rank) or grew
        if full:
            converged = _check(sk, sk.cores(), rng, GATE)[0][0] <= thr
            break
        if swe <= thr:
            clean += 1
            if clean >= 2:
                gate = _check(sk, sk.cores(), rng, GATE, top=INJECT)
                if gate[0][0] <= thr:
                    converged = True
                    break
                clean = 0
                grew = _inject(sk, gate, thr, max_rank) or grew
        else:
            clean = 0
        if not grew and clean == 0:
            break

    final = sk.cores()
    vp = rng.integers(0, shape, size=(validation_count, d))
    vref = memo(vp)

    def validate(c):
        e = float(np.max(np.abs(vref - at_indices(c, vp))))
        return max(e, _check(sk, c, rng, GATE)[0][0])

    achieved = validate(final)
    if best is not None and best_err < achieved:
        alt = validate(best)
        if alt < achieved:
            final, achieved = best, alt
    achieved /= max(memo.max_abs, TINY)
    return CrossOut([np.array(c, dtype=np.float64) for c in final], achieved,
                    memo.calls, sweeps, converged)
