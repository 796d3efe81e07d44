"""TEST-ONLY CPU stand-in for distributed.CudaShard: the same per-shard math
(K1 / K2 / finalize of k_spmv.cu) on numpy, over the oracle's rows / columns,
so the distributed driver's host logic (partition, halo windows, exchange
pattern, scalar all-reduce, stop handling) runs under gloo on CPU."""
import math

import numpy as np
import torch

from paper_1503_03520_b200.distributed import partition


class CpuShard:
    def __init__(self, oracle, inst, rank, world, max_iters):
        self.rank, self.world, self.single = rank, world, False
        n = inst.n
        h = (len(inst.op.right_offset) + 1) & ~1  # window overhang: #stages rounded up to even
        a, b = partition(n, world)[rank]
        self.own, self.halo, self.a = b - a, h, a
        rp, ri, rv = oracle.csr(inst.op)
        cp, ci, cv = oracle.csc(inst.op)
        base = a - h
        self.rows = [(ri[rp[i]:rp[i + 1]].astype(np.int64) - base, rv[rp[i]:rp[i + 1]]) for i in range(a, b)]
        self.cols = [(ci[cp[j]:cp[j + 1]].astype(np.int64) - base, cv[cp[j]:cp[j + 1]]) for j in range(a, b)]
        W = self.own + 2 * h
        self.x_win = torch.zeros(W, dtype=torch.float64)
        self.r_y_win = torch.zeros(W, dtype=torch.float64)
        self.scal = torch.zeros(4, dtype=torch.float64)
        self.y = np.zeros(self.own)
        self.b = inst.b[a:b].copy()
        self.r_x = 0.0 - self.b
        self.r_y_win[h:h + self.own] = torch.from_numpy(self.r_x.copy())
        self.scal[3] = float(np.sum(self.r_x * self.r_x))
        self.tau, self.L = inst.tau, oracle.gram_lmax(inst.op)
        self.t, self.k, self.stop, self.init = 1.0, 0, False, False
        self.max_iters = max_iters
        self.samples = []

    def _beta(self):
        t_next = 0.5 * (1.0 + math.sqrt(1.0 + 4.0 * self.t * self.t))
        return t_next, (self.t - 1.0) / t_next

    def k1(self):
        if self.stop:
            return
        h, r = self.halo, self.r_y_win.numpy()
        x = self.x_win.numpy()
        _, beta = self._beta()
        inv_l = 1.0 / self.L
        l1 = nnz = mism = 0.0
        for j, (idx, val) in enumerate(self.cols):
            g = 0.0
            for q in range(len(idx)):
                g += val[q] * r[idx[q]]
            yo, xo = self.y[j], x[h + j]
            v = yo - inv_l * g
            thr = self.tau * inv_l
            tr = v - thr if v > thr else (v + thr if v < -thr else 0.0)
            mism += tr != yo
            self.y[j] = tr + beta * (tr - xo)
            x[h + j] = tr
            l1 += abs(tr)
            nnz += tr != 0.0
        self.scal[0], self.scal[1], self.scal[2] = l1, nnz, mism

    def k2(self):
        if self.stop:
            return
        h, x = self.halo, self.x_win.numpy()
        ry = self.r_y_win.numpy()
        _, beta = self._beta()
        rr = 0.0
        for i, (idx, val) in enumerate(self.rows):
            s = 0.0
            for q in range(len(idx)):
                s += val[q] * x[idx[q]]
            rt = s - self.b[i]
            ry[h + i] = (1.0 + beta) * rt - beta * self.r_x[i]
            self.r_x[i] = rt
            rr += rt * rt
        self.scal[3] = rr

    def finalize(self):
        if self.stop:
            return
        sc = self.scal.numpy()
        if not self.init:
            self.init = True
            f = 0.5 * sc[3]
            self.samples.append((0, f))
            self.stop = self.max_iters == 0
            return
        f = self.tau * sc[0] + 0.5 * sc[3]
        t_next, _ = self._beta()
        self.t = t_next
        self.k += 1
        self.samples.append((self.k, f))
        if sc[2] == 0.0 or self.k >= self.max_iters:
            self.stop = True

    def stopped(self):
        return self.stop, self.k

    def finish(self):
        return self.samples, self.x_win.numpy()[self.halo:self.halo + self.own].copy()


class CpuShardSingle:
    """Single-kernel mode stand-in (k_fused.cu fista_iter_kernel): x / r rotate
    through three halo windows; y and r_y are formed from the last two
    iterates; after each iteration the caller exchanges the halos of the new
    x (H) and r (2H) windows."""

    def __init__(self, oracle, inst, rank, world, max_iters):
        self.rank, self.world, self.single = rank, world, True
        n = inst.n
        H = (len(inst.op.right_offset) + 1) & ~1
        a, b = partition(n, world)[rank]
        self.n, self.a, self.b_, self.own = n, a, b, b - a
        self.x_halo, self.r_halo = H, 2 * H
        rp, ri, rv = oracle.csr(inst.op)
        cp, ci, cv = oracle.csc(inst.op)
        # columns of the x window [a - H, b + H) with rows local to the r window [a - 2H, ...)
        self.cols = {}
        for j in range(max(0, a - H), min(n, b + H)):
            self.cols[j] = (ci[cp[j]:cp[j + 1]].astype(np.int64) - (a - 2 * H), cv[cp[j]:cp[j + 1]])
        self.rows = [(ri[rp[i]:rp[i + 1]].astype(np.int64) - (a - H), rv[rp[i]:rp[i + 1]]) for i in range(a, b)]
        self.x_bufs = [torch.zeros(self.own + 2 * H, dtype=torch.float64) for _ in range(3)]
        self.r_bufs = [torch.zeros(self.own + 4 * H, dtype=torch.float64) for _ in range(3)]
        self.b = inst.b[a:b].copy()
        r0 = 0.0 - self.b
        for q in (0, 2):
            self.r_bufs[q][2 * H:2 * H + self.own] = torch.from_numpy(r0.copy())
        self.scal = torch.zeros(4, dtype=torch.float64)
        self.scal[3] = float(np.sum(r0 * r0))
        self.tau, self.L = inst.tau, oracle.gram_lmax(inst.op)
        self.t, self.beta_y, self.k, self.j = 1.0, 0.0, 0, 0
        self.stop, self.init = False, False
        self.max_iters = max_iters
        self.samples = []

    def next_halos(self):
        q = self.j % 3
        return [(self.x_bufs[q], self.x_halo), (self.r_bufs[q], self.r_halo)]

    def initial_halos(self):
        return [(self.r_bufs[0], self.r_halo), (self.r_bufs[2], self.r_halo)]

    def k1(self):
        j, self.j = self.j, self.j + 1
        if self.stop:
            return
        H, a, n, beta = self.x_halo, self.a, self.n, self.beta_y
        xk, xkm1 = self.x_bufs[j % 3].numpy(), self.x_bufs[(j + 2) % 3].numpy()
        rk, rkm1 = self.r_bufs[j % 3].numpy(), self.r_bufs[(j + 2) % 3].numpy()
        xn, rn = self.x_bufs[(j + 1) % 3].numpy(), self.r_bufs[(j + 1) % 3].numpy()
        ry = (1.0 + beta) * rk - beta * rkm1
        inv_l = 1.0 / self.L
        thr = self.tau * inv_l
        trial = np.zeros(self.own + 2 * H)
        l1 = nnz = mism = 0.0
        for jj, (idx, val) in self.cols.items():
            g = 0.0
            for q in range(len(idx)):
                g += val[q] * ry[idx[q]]
            lx = jj - (a - H)
            y = xk[lx] + beta * (xk[lx] - xkm1[lx])
            v = y - inv_l * g
            tr = v - thr if v > thr else (v + thr if v < -thr else 0.0)
            trial[lx] = tr
            if a <= jj < self.b_:
                xn[lx] = tr
                l1 += abs(tr)
                nnz += tr != 0.0
                mism += tr != y
        rr = 0.0
        for i, (idx, val) in enumerate(self.rows):
            s = 0.0
            for q in range(len(idx)):
                s += val[q] * trial[idx[q]]
            rt = s - self.b[i]
            rn[2 * H + i] = rt
            rr += rt * rt
        self.scal[0], self.scal[1], self.scal[2], self.scal[3] = l1, nnz, mism, rr

    def k2(self):
        pass

    def finalize(self):
        if self.stop:
            return
        sc = self.scal.numpy()
        if not self.init:
            self.init = True
            self.samples.append((0, 0.5 * sc[3]))
            self.stop = self.max_iters == 0
            return
        f = self.tau * sc[0] + 0.5 * sc[3]
        t_next = 0.5 * (1.0 + math.sqrt(1.0 + 4.0 * self.t * self.t))
        self.beta_y = (self.t - 1.0) / t_next
        self.t = t_next
        self.k += 1
        self.samples.append((self.k, f))
        if sc[2] == 0.0 or self.k >= self.max_iters:
            self.stop = True

    def stopped(self):
        return self.stop, self.k

    def finish(self):
        q = self.k % 3
        return self.samples, self.x_bufs[q].numpy()[self.x_halo:self.x_halo + self.own].copy()


class CpuShardRc:
    """Recomputing-kernel stand-in (k_iter_rc.cu fista_rc_kernel): only x
    travels (three windows with halo H3 = 2S rounded up to 4); r_k, r_{k-1}
    are rebuilt from x_k, x_{k-1} on the rows around the block (b window);
    scal[3] is ||r_k||^2 of the iterate the kernel started from, so the
    objective of iteration j is recorded by the finalize after kernel j
    (fista_finalize_lagged) and a flush records the last one."""

    def __init__(self, oracle, inst, rank, world, max_iters):
        self.rank, self.world, self.single, self.lagged = rank, world, True, True
        n = inst.n
        S = len(inst.op.right_offset)
        H3 = (2 * S + 3) // 4 * 4
        a, b = partition(n, world)[rank]
        self.n, self.a, self.b_, self.own, self.S = n, a, b, b - a, S
        self.x_halo, self.r_halo = H3, 0
        rp, ri, rv = oracle.csr(inst.op)
        cp, ci, cv = oracle.csc(inst.op)
        base = a - H3  # window-local index of global entry g: g - base
        # rows [a - S, b + S) over the x window; columns [a, b) over those rows
        self.rlo, self.rhi = max(0, a - S), min(n, b + S)
        self.rows = {i: (ri[rp[i]:rp[i + 1]].astype(np.int64) - base, rv[rp[i]:rp[i + 1]])
                     for i in range(self.rlo, self.rhi)}
        self.cols = [(ci[cp[j]:cp[j + 1]].astype(np.int64), cv[cp[j]:cp[j + 1]]) for j in range(a, b)]
        self.bwin = {i: inst.b[i] for i in range(self.rlo, self.rhi)}
        self.x_bufs = [torch.zeros(self.own + 2 * H3, dtype=torch.float64) for _ in range(3)]
        self.r_bufs = None
        self.scal = torch.zeros(4, dtype=torch.float64)
        self.scal[3] = float(sum((0.0 - inst.b[i]) ** 2 for i in range(a, b)))
        self.tau, self.L = inst.tau, oracle.gram_lmax(inst.op)
        self.t, self.beta_y, self.k, self.j = 1.0, 0.0, 0, 0
        self.stop, self.init, self.pend, self.flushing = False, False, None, False
        self.max_iters = max_iters
        self.samples = []

    def next_halos(self):
        return [(self.x_bufs[self.j % 3], self.x_halo)]

    def initial_halos(self):
        return []

    def _r(self, x):
        return {i: sum(v * x[q] for q, v in zip(*self.rows[i])) - self.bwin[i] for i in self.rows}

    def k1(self, flush=False):
        j = self.j
        if not flush:
            self.j += 1
        if self.stop:
            return
        H, a, beta = self.x_halo, self.a, self.beta_y
        xk, xkm1 = self.x_bufs[j % 3].numpy(), self.x_bufs[(j + 2) % 3].numpy()
        rk = self._r(xk)
        rr = sum(rk[i] ** 2 for i in range(a, self.b_))
        if flush:
            self.flushing = True
            self.scal[0], self.scal[1], self.scal[2], self.scal[3] = 0.0, 0.0, 0.0, rr
            return
        rkm1 = self._r(xkm1)
        xn = self.x_bufs[(j + 1) % 3].numpy()
        inv_l = 1.0 / self.L
        thr = self.tau * inv_l
        l1 = nnz = mism = 0.0
        for jj, (idx, val) in zip(range(a, self.b_), self.cols):
            g = sum(v * ((1.0 + beta) * rk[i] - beta * rkm1[i]) for i, v in zip(idx, val))
            lx = jj - (a - H)
            y = xk[lx] + beta * (xk[lx] - xkm1[lx])
            v = y - inv_l * g
            tr = v - thr if v > thr else (v + thr if v < -thr else 0.0)
            xn[lx] = tr
            l1 += abs(tr)
            nnz += tr != 0.0
            mism += tr != y
        self.scal[0], self.scal[1], self.scal[2], self.scal[3] = l1, nnz, mism, rr

    def k2(self):
        pass

    def flush(self):
        self.k1(flush=True)

    def finalize(self):
        if self.stop:
            return
        sc = self.scal.numpy().copy()
        if not self.init:
            self.init = True
            self.samples.append((0, 0.5 * sc[3]))
            self.stop = self.max_iters == 0
            return
        if self.pend is not None:
            l1, _, mism = self.pend
            self.pend = None
            self.k += 1
            self.samples.append((self.k, self.tau * l1 + 0.5 * sc[3]))
            if mism == 0.0 or self.k >= self.max_iters:
                self.stop = True
                return
        if self.flushing:
            return
        t_next = 0.5 * (1.0 + math.sqrt(1.0 + 4.0 * self.t * self.t))
        self.beta_y = (self.t - 1.0) / t_next
        self.t = t_next
        self.pend = (sc[0], sc[1], sc[2])

    def stopped(self):
        return self.stop, self.k

    def finish(self):
        q = self.k % 3
        return self.samples, self.x_bufs[q].numpy()[self.x_halo:self.x_halo + self.own].copy()


class CpuShardRc2:
    """Two-iterations-per-launch stand-in (k_iter_rc.cu fista_rc2v_kernel, the
    default shard mode): x rotates through four windows with halo H = 4S; one
    k1() rebuilds r_j, r_{j-1} on rows [a-3S, b+3S), forms x_{j+1} on columns
    [a-2S, b+2S), r_{j+1} on rows [a-S, b+S) and x_{j+2} on the own columns,
    and leaves the 8 sums of scal8 (||r_j||^2, l1 / nnz / mismatches of
    x_{j+1}, ||r_{j+1}||^2, those of x_{j+2}) for the all-reduce; finalize
    records two iterations (fista_finalize_lagged2); the flush records the
    last iterate (fista_finalize_lagged)."""

    def __init__(self, oracle, inst, rank, world, max_iters):
        self.rank, self.world, self.single, self.lagged, self.pairs = rank, world, True, True, True
        n = inst.n
        S = len(inst.op.right_offset)
        H = 4 * S
        a, b = partition(n, world)[rank]
        self.n, self.a, self.b_, self.own, self.S = n, a, b, b - a, S
        self.x_halo, self.r_halo, self.nbuf = H, 0, 4
        rp, ri, rv = oracle.csr(inst.op)
        cp, ci, cv = oracle.csc(inst.op)
        base = a - H  # window-local index of global entry g: g - base
        self.base = base
        self.rows = {i: (ri[rp[i]:rp[i + 1]].astype(np.int64) - base, rv[rp[i]:rp[i + 1]])
                     for i in range(max(0, a - 3 * S), min(n, b + 3 * S))}
        self.cols = {j: (ci[cp[j]:cp[j + 1]].astype(np.int64), cv[cp[j]:cp[j + 1]])
                     for j in range(max(0, a - 2 * S), min(n, b + 2 * S))}
        self.bwin = {i: inst.b[i] for i in self.rows}
        self.x_bufs = [torch.zeros(self.own + 2 * H, dtype=torch.float64) for _ in range(4)]
        self.r_bufs = None
        self.scal = torch.zeros(4, dtype=torch.float64)
        self.scal8 = torch.zeros(8, dtype=torch.float64)
        self.scal[3] = float(sum((0.0 - inst.b[i]) ** 2 for i in range(a, b)))
        self.scal_now = self.scal
        self.tau, self.L = inst.tau, oracle.gram_lmax(inst.op)
        self.t, self.beta_y, self.k, self.j = 1.0, 0.0, 0, 0
        self.stop, self.init, self.pend, self.flushing = False, False, None, False
        self.max_iters = max_iters
        self.samples = []

    def next_halos(self):  # x_{j-1} and x_j were both written
        return [(self.x_bufs[(self.j - 1) % 4], self.x_halo), (self.x_bufs[self.j % 4], self.x_halo)]

    def initial_halos(self):
        return []

    def _r(self, x, lo, hi):
        return {i: sum(v * x[q] for q, v in zip(*self.rows[i])) - self.bwin[i]
                for i in range(max(0, lo), min(self.n, hi))}

    def _momentum(self):
        t_next = 0.5 * (1.0 + math.sqrt(1.0 + 4.0 * self.t * self.t))
        return t_next, (self.t - 1.0) / t_next

    def _prox(self, xk, xm, r1, r0, beta, lo, hi, out):
        """x_new on columns [lo, hi) from x_k, x_{k-1} (windows) and the
        residuals r1 = r_k, r0 = r_{k-1}; returns the own-column sums."""
        inv_l = 1.0 / self.L
        thr = self.tau * inv_l
        l1 = nnz = mism = 0.0
        for jj in range(max(0, lo), min(self.n, hi)):
            idx, val = self.cols[jj]
            g = sum(v * ((1.0 + beta) * r1[i] - beta * r0[i]) for i, v in zip(idx, val))
            lx = jj - self.base
            y = xk[lx] + beta * (xk[lx] - xm[lx])
            v = y - inv_l * g
            tr = v - thr if v > thr else (v + thr if v < -thr else 0.0)
            out[lx] = tr
            if self.a <= jj < self.b_:
                l1 += abs(tr)
                nnz += tr != 0.0
                mism += tr != y
        return l1, nnz, mism

    def k1(self):
        j, S, a, b = self.j, self.S, self.a, self.b_
        self.j += 2
        self.scal_now = self.scal8
        if self.stop:
            return
        xk, xm = self.x_bufs[j % 4].numpy(), self.x_bufs[(j + 3) % 4].numpy()
        t_next, beta_b = self._momentum()
        rk = self._r(xk, a - 3 * S, b + 3 * S)
        rm = self._r(xm, a - 3 * S, b + 3 * S)
        rr0 = sum(rk[i] ** 2 for i in range(a, b))
        x1 = np.zeros_like(xk)
        l1a, nza, misa = self._prox(xk, xm, rk, rm, self.beta_y, a - 2 * S, b + 2 * S, x1)
        r1 = self._r(x1, a - S, b + S)
        rr1 = sum(r1[i] ** 2 for i in range(a, b))
        x2 = np.zeros_like(xk)
        l1b, nzb, misb = self._prox(x1, xk, r1, rk, beta_b, a, b, x2)
        H, own = self.x_halo, self.own
        self.x_bufs[(j + 1) % 4].numpy()[H:H + own] = x1[H:H + own]
        self.x_bufs[(j + 2) % 4].numpy()[H:H + own] = x2[H:H + own]
        self.scal8[:] = torch.tensor([rr0, l1a, nza, misa, rr1, l1b, nzb, misb], dtype=torch.float64)

    def k2(self):
        pass

    def flush(self):  # ||r||^2 of the newest iterate, recorded by a lagged finalize
        self.scal_now = self.scal
        if self.stop:
            return
        x = self.x_bufs[self.j % 4].numpy()
        r = self._r(x, self.a, self.b_)
        self.scal[0], self.scal[1], self.scal[2] = 0.0, 0.0, 0.0
        self.scal[3] = sum(r[i] ** 2 for i in range(self.a, self.b_))
        self.flushing = True

    def _record(self, f, mism):
        self.k += 1
        self.samples.append((self.k, f))
        if mism == 0.0 or self.k >= self.max_iters:
            self.stop = True

    def finalize(self):
        if self.stop:
            return
        if not self.init:
            self.init = True
            self.samples.append((0, 0.5 * float(self.scal[3])))
            self.stop = self.max_iters == 0
            return
        if self.flushing:  # fista_finalize_lagged(flush)
            if self.pend is not None:
                l1, _, mism = self.pend
                self.pend = None
                self._record(self.tau * l1 + 0.5 * float(self.scal[3]), mism)
            return
        q = self.scal8.numpy().copy()
        if self.pend is not None:  # iteration j: stashed sums + ||r_j||^2
            l1, _, mism = self.pend
            self.pend = None
            self._record(self.tau * l1 + 0.5 * q[0], mism)
            if self.stop:
                return
        self.t, self.beta_y = self._momentum()  # the step the kernel used for x_{j+2}
        self._record(self.tau * q[1] + 0.5 * q[4], q[3])  # iteration j+1
        if self.stop:
            return
        self.t, self.beta_y = self._momentum()
        self.pend = (q[5], q[6], q[7])

    def stopped(self):
        return self.stop, self.k

    def finish(self):
        q = self.k % 4
        return self.samples, self.x_bufs[q].numpy()[self.x_halo:self.x_halo + self.own].copy()


class CpuShardGeneral:
    """General-operator stand-in (permuted rows): rows [a, b) of A (CSR, global
    columns) and the CSC of that block; x split by columns in slices of cs
    (n_pad = world * cs); the driver reduce-scatters g_full and all-gathers
    x_full (distributed.reduce_scatter_slices / all_gather_slices)."""

    def __init__(self, oracle, inst, rank, world, max_iters):
        self.rank, self.world, self.single, self.lagged, self.general = rank, world, False, False, True
        n, m = inst.n, len(inst.b)
        cut = lambda q: m if q == world else (m * q // world) // 16 * 16  # noqa: E731
        a, b = cut(rank), cut(rank + 1)
        cs = ((n + world - 1) // world + 15) // 16 * 16
        self.n, self.a, self.b_, self.cs = n, a, b, cs
        self.n_pad = world * cs
        self.col_begin = rank * cs
        self.col_count = max(0, min(n, (rank + 1) * cs) - min(n, rank * cs))
        rp, ri, rv = oracle.csr(inst.op)
        cp, ci, cv = oracle.csc(inst.op)
        nrow = len(rp) - 1
        self.rows = [(ri[rp[i]:rp[i + 1]].astype(np.int64), rv[rp[i]:rp[i + 1]]) if i < nrow else
                     (np.zeros(0, np.int64), np.zeros(0)) for i in range(a, b)]
        self.cols = []
        for j in range(n):
            idx, val = ci[cp[j]:cp[j + 1]].astype(np.int64), cv[cp[j]:cp[j + 1]]
            keep = (idx >= a) & (idx < b)
            self.cols.append((idx[keep] - a, val[keep]))
        self.g_full = torch.zeros(self.n_pad, dtype=torch.float64)
        self.x_full = torch.zeros(self.n_pad, dtype=torch.float64)
        self.y = np.zeros(cs)
        self.bown = inst.b[a:b].copy()
        self.r_x = 0.0 - self.bown
        self.r_y = self.r_x.copy()
        self.scal = torch.zeros(4, dtype=torch.float64)
        self.scal[3] = float(np.sum(self.r_x * self.r_x))
        self.tau, self.L = inst.tau, oracle.gram_lmax(inst.op)
        self.t, self.k, self.stop, self.init = 1.0, 0, False, False
        self.max_iters = max_iters
        self.samples = []

    def _beta(self):
        t_next = 0.5 * (1.0 + math.sqrt(1.0 + 4.0 * self.t * self.t))
        return t_next, (self.t - 1.0) / t_next

    def k1(self):
        if self.stop:
            return
        g = self.g_full.numpy()
        g[:] = 0.0
        for j, (idx, val) in enumerate(self.cols):
            s = 0.0
            for q in range(len(idx)):
                s += val[q] * self.r_y[idx[q]]
            g[j] = s

    def prox(self):
        if self.stop:
            return
        g, x = self.g_full.numpy(), self.x_full.numpy()
        _, beta = self._beta()
        inv_l = 1.0 / self.L
        thr = self.tau * inv_l
        l1 = nnz = mism = 0.0
        for q in range(self.col_count):
            j = self.col_begin + q
            yo, xo = self.y[q], x[j]
            v = yo - inv_l * g[j]
            tr = v - thr if v > thr else (v + thr if v < -thr else 0.0)
            mism += tr != yo
            self.y[q] = tr + beta * (tr - xo)
            x[j] = tr
            l1 += abs(tr)
            nnz += tr != 0.0
        self.scal[0], self.scal[1], self.scal[2] = l1, nnz, mism

    def k2(self):
        if self.stop:
            return
        x = self.x_full.numpy()
        _, beta = self._beta()
        rr = 0.0
        for i, (idx, val) in enumerate(self.rows):
            s = 0.0
            for q in range(len(idx)):
                s += val[q] * x[idx[q]]
            rt = s - self.bown[i]
            self.r_y[i] = (1.0 + beta) * rt - beta * self.r_x[i]
            self.r_x[i] = rt
            rr += rt * rt
        self.scal[3] = rr

    def finalize(self):
        if self.stop:
            return
        sc = self.scal.numpy()
        if not self.init:
            self.init = True
            self.samples.append((0, 0.5 * sc[3]))
            self.stop = self.max_iters == 0
            return
        f = self.tau * sc[0] + 0.5 * sc[3]
        t_next, _ = self._beta()
        self.t = t_next
        self.k += 1
        self.samples.append((self.k, f))
        if sc[2] == 0.0 or self.k >= self.max_iters:
            self.stop = True

    def stopped(self):
        return self.stop, self.k

    def finish(self):
        x = self.x_full.numpy()
        return self.samples, x[self.col_begin:self.col_begin + self.col_count].copy()
