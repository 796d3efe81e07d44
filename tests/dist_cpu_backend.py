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
        self.rank, self.world = rank, world
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
