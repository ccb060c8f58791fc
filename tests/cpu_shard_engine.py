"""Oracle-backed CPU implementation of the shard-engine protocol of
paper_1204_0069_b200.sharded (TEST INFRASTRUCTURE).

Each phase does what the CUDA library's phase does (include/coopcg_gpu.h),
with the reference's arithmetic (ascending sequential dots via the C oracle,
kernels.hpp:20-49; LU via the oracle, kernels.hpp:61-115), on row-sharded A
and replicated torch CPU blocks, so that tests/test_sharded_gloo.py can run the
real orchestrator and its gloo all-gathers in two processes and compare with
an unsharded oracle solve bit for bit.
"""
import contextlib
import ctypes as C
import math
from types import SimpleNamespace

import numpy as np
import torch

import pyoracle as po
from paper_1204_0069_b200.sharded import (BLOCK_D, BLOCK_Q, BLOCK_R, BLOCK_S, BLOCK_X, PH_FINAL_LOCAL,
                                          PH_FINAL_REST, PH_ITER_LOCAL, PH_ITER_MID, PH_ITER_REST,
                                          PH_MCCG_SETUP, PH_SETUP_LOCAL, PH_SETUP_REST, row_split)


def _dot(a, b):
    a = np.ascontiguousarray(a)
    b = np.ascontiguousarray(b)
    return po.oracle_lib().orc_dot(a.ctypes.data, b.ctypes.data, len(a))


def _combine(base, B, coeff):
    acc = base.copy()
    for j in range(len(coeff)):
        acc = acc + coeff[j] * B[:, j]
    return acc


class CpuShardEngine:
    def __init__(self, A, b, X0, rank, world):
        self.A = np.ascontiguousarray(A)
        self.b = np.ascontiguousarray(b)
        self.n, self.p = X0.shape
        self.P = self.p0 = self.p
        self.X0 = np.array(X0, dtype=np.float64)
        self.row0, self.row1, _ = row_split(self.n, world, rank)
        z = lambda: torch.zeros((self.n, self.P), dtype=torch.float64)
        self.X = torch.from_numpy(np.array(X0, dtype=np.float64))
        self.R, self.Q, self.S = z(), z(), z()
        self.Dblk = [z(), z()]

    # -- protocol --
    def collective_stream(self):
        return contextlib.nullcontext()

    def block(self, which, k):
        return {BLOCK_X: self.X, BLOCK_R: self.R, BLOCK_D: self.Dblk[k & 1], BLOCK_Q: self.Q,
                BLOCK_S: self.S}[which]

    def begin(self, opts):
        self.tol = opts.tol
        self.max_iters = opts.max_iters if opts.max_iters >= 0 else 2 * self.n
        self.every = opts.recompute_residual_every if opts.recompute_residual_every >= 0 else 50
        self.rank_tol = opts.rank_rel_tol
        self.stop, self.status, self.k, self.err = False, "max-iterations", 0, None
        self.converged_agent = -1
        self.records = []
        # mccg_solve (solvers.hpp:338-342): agents restricted on rank drops
        self.mccg = opts.algo == "mccg"
        self.p = self.p0
        self.ids = list(range(self.p0))
        self.pending = None
        self.X.copy_(torch.from_numpy(self.X0))

    def recompute_at(self, k):
        return self.every > 0 and (k + 1) % self.every == 0

    def state(self):
        return self.stop, len(self.records)

    def _local_residual(self, dst):
        Xn = self.X.numpy()
        for i in range(self.row0, self.row1):
            for j in range(self.p):
                dst[i, j] = _dot(self.A[i], Xn[:, j]) - self.b[i]

    def _first_converged(self, norms):
        for j, v in enumerate(norms):
            if v <= self.tol:
                return j
        return -1

    def phase(self, ph, k):
        n, p = self.n, self.p
        if ph == PH_SETUP_LOCAL:
            self._local_residual(self.R.numpy())
        elif ph == PH_SETUP_REST:
            self.Dblk[0].copy_(self.R)
            Rn = self.R.numpy()
            self.norms = [math.sqrt(_dot(Rn[:, j], Rn[:, j])) for j in range(p)]
            self.initial = list(self.norms)
            rank0, cols = po.numerical_rank(self.Dblk[0].numpy(), self.rank_tol)
            if self.mccg and 0 < rank0 < p:  # setup_coordinator's restriction (solvers.hpp:63-76)
                self._restrict(sorted(int(c) for c in cols), self.Dblk[0])
                Rn = self.R.numpy()
                self.norms = [math.sqrt(_dot(Rn[:, j], Rn[:, j])) for j in range(self.p)]
            slot = self._first_converged(self.norms)
            if slot >= 0:
                self.stop, self.status, self.converged_agent = True, "converged", self.ids[slot]
            elif not self.mccg and rank0 < p:
                self.stop, self.status = True, "rank-collapse"
            elif self.mccg and rank0 == 0:
                self.err, self.stop = "every starting direction is numerically zero", True
            if not self.stop and self.max_iters == 0:
                self.stop = True
        elif ph == PH_MCCG_SETUP:
            pass  # done with SETUP_REST above
        elif ph in (PH_ITER_LOCAL, PH_ITER_MID, PH_ITER_REST):
            if self.stop:
                return
            D = self.Dblk[k & 1].numpy()
            Dn = self.Dblk[(k + 1) & 1].numpy()
            Qn, Rn, Xn = self.Q.numpy(), self.R.numpy(), self.X.numpy()
            if ph == PH_ITER_LOCAL:
                for i in range(self.row0, self.row1):
                    for j in range(p):
                        Qn[i, j] = _dot(self.A[i], D[:, j])
            elif ph == PH_ITER_MID:
                raw = np.array([[_dot(D[:, i], Qn[:, j]) for j in range(p)] for i in range(p)])
                self.M = (raw + raw.T) / 2.0
                for i in range(p):
                    if not (self.M[i, i] > 0.0) and _dot(D[:, i], D[:, i]) > 0.0:
                        self.err, self.stop = f"nonpositive direction energy d^T A d at iteration {k}", True
                        return
                rhs = np.array([[-_dot(Rn[:, i], D[:, j]) for j in range(p)] for i in range(p)])
                self.lu, self.perm, ok = self._lu(self.M)
                if not ok:
                    self.stop, self.status = True, "rank-collapse"
                    return
                alpha = np.array([self._lu_solve(rhs[i]) for i in range(p)])
                rec = self.recompute_at(k)
                for i in range(p):
                    if not rec:
                        Rn[:, i] = _combine(Rn[:, i], Qn, alpha[i])
                    Xn[:, i] = _combine(Xn[:, i], D, alpha[i])
                if rec:
                    self._local_residual(Rn)
            else:
                rhs = np.array([[-_dot(Rn[:, i], Qn[:, j]) for j in range(p)] for i in range(p)])
                beta = np.array([self._lu_solve(rhs[i]) for i in range(p)])
                for i in range(p):
                    Dn[:, i] = _combine(Rn[:, i], D, beta[i])
                norms = [math.sqrt(_dot(Rn[:, j], Rn[:, j])) for j in range(p)]
                m = norms[0]
                for v in norms:
                    m = v if v < m else m
                row = [math.nan] * self.p0  # per original agent id (IterationRecord::agents)
                for j in range(p):
                    row[self.ids[j]] = norms[j]
                self.records.append((row, m))
                slot = self._first_converged(norms)
                rr = -1
                if slot < 0:
                    rr = po.numerical_rank(Dn[:, :p], self.rank_tol)[0]
                if slot >= 0:
                    self.stop, self.status, self.converged_agent = True, "converged", self.ids[slot]
                elif rr < p and self.mccg:  # pause for the restriction (mccg_resume)
                    self.stop, self.pending = True, (k, rr)
                elif rr < p:
                    self.stop, self.status = True, "rank-collapse"
                elif k + 1 >= self.max_iters:
                    self.stop, self.status = True, "max-iterations"
        elif ph == PH_FINAL_LOCAL:
            self._local_residual(self.S.numpy())
        elif ph == PH_FINAL_REST:
            Sn = self.S.numpy()
            self.final = [math.nan] * self.p0
            for j in range(p):
                self.final[self.ids[j]] = math.sqrt(_dot(Sn[:, j], Sn[:, j]))

    def _restrict(self, keep, direction):
        """BlockCgWorkspace::restrict_to (block_cg.hpp:84-96) on the replicated blocks."""
        for blk in (self.X, self.R, direction):
            a = blk.numpy()
            kept = a[:, keep].copy()
            a[:, :] = 0.0
            a[:, :len(keep)] = kept
        self.ids = [self.ids[c] for c in keep]
        self.p = len(keep)

    def mccg_resume(self):
        """end_of_iteration's restriction (solvers.hpp:156-175) after a paused rank drop."""
        if not self.pending:
            return -1
        k, rr = self.pending
        self.pending = None
        nsel, cols = po.numerical_rank(self.R.numpy()[:, :self.p], self.rank_tol)
        pnext = min(rr, nsel)
        if pnext == 0:
            self.err = f"all agents degenerate at iteration {k} with residual above tolerance"
            return -1
        self._restrict(sorted(int(c) for c in cols[:pnext]), self.Dblk[(k + 1) & 1])
        if k + 1 >= self.max_iters:
            self.status = "max-iterations"
            return -1
        self.stop = False
        return k + 1

    def _lu(self, M):
        p = self.p
        lu = np.ascontiguousarray(M.copy())
        perm = np.zeros(p, dtype=np.int32)
        maxabs = 0.0
        for v in M.ravel():
            maxabs = abs(v) if maxabs < abs(v) else maxabs
        ok = po.oracle_lib().orc_lu_factor(lu.ctypes.data_as(C.c_void_p), p, perm.ctypes.data_as(C.c_void_p),
                                           C.c_double(maxabs * 1e-14))
        return lu, perm, bool(ok)

    def _lu_solve(self, rhs):
        rhs = np.ascontiguousarray(rhs)
        x = np.zeros(self.p)
        po.oracle_lib().orc_lu_solve_vec(self.lu.ctypes.data_as(C.c_void_p), self.p,
                                         self.perm.ctypes.data_as(C.c_void_p), rhs.ctypes.data_as(C.c_void_p),
                                         x.ctypes.data_as(C.c_void_p))
        return x

    def end(self):
        if self.err:
            raise RuntimeError(self.err)
        return SimpleNamespace(status=self.status, iterations=len(self.records), converged_agent=self.converged_agent,
                               residual_norms=np.array([r[0] for r in self.records]).reshape(-1, self.p0),
                               minres=np.array([r[1] for r in self.records]),
                               final_x=self.X.numpy()[:, :self.p].copy(), active_agents=list(self.ids),
                               final_residual_norms=np.array(self.final), initial=np.array(self.initial))
