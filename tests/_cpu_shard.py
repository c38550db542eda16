"""CPU stand-in for one libdit shard (test infrastructure, not product code).

Implements the di_shard_* protocol of include/dit.h with plain numpy float64
arithmetic (the frontier sweep of DESIGN.md reading R1 restricted to owned
nodes, remote pushes into ghost slots), so that the multi-rank host logic in
paper_1501_06350_b200/dist.py can be exercised with the gloo backend on CPU.
"""
import numpy as np
import torch


class CpuShard:
    def __init__(self, n_global, lo, hi, row_ptr, col, weights=None):
        self.n_global, self.lo, self.hi = int(n_global), int(lo), int(hi)
        self.n_local = hi - lo
        col = np.asarray(col, dtype=np.int64)
        remote = (col < lo) | (col >= hi)
        gids = np.unique(col[remote])
        self.n_ghost = len(gids)
        self.ghost_ids = torch.tensor(gids.astype(np.int32))
        slot = np.where(remote, self.n_local + np.searchsorted(gids, col), col - lo)
        self.row_ptr = np.asarray(row_ptr, dtype=np.int64)
        self.slot = slot
        deg = np.diff(self.row_ptr)
        w = np.ones(len(col)) if weights is None else np.asarray(weights, dtype=np.float64)
        src = np.repeat(np.arange(self.n_local), deg)
        wsum = np.bincount(src, weights=w, minlength=self.n_local)
        self.p = np.where(deg[src] > 0, w / np.where(wsum[src] > 0, wsum[src], 1.0), 0.0)
        self.src = src
        self.deg = deg
        self.send = torch.zeros(max(self.n_ghost, 1), dtype=torch.float64)
        self.stats = torch.zeros(4, dtype=torch.float64)
        self.gathered = torch.zeros(4, dtype=torch.float64)
        self.world = 1
        self.recv = torch.zeros(1, dtype=torch.float64)
        self.send_counts = self.recv_counts = None

    def set_recv(self, local_idx, seg_counts):
        self.recv_idx = np.asarray(local_idx, dtype=np.int64)
        self.recv_counts = [int(c) for c in seg_counts]
        self.world = len(self.recv_counts)
        self.gathered = torch.zeros(4 * self.world, dtype=torch.float64)
        self.recv = torch.zeros(max(sum(self.recv_counts), 1), dtype=torch.float64)

    def begin(self, d, tol, theta=1.0, max_sweeps=0, **_):
        self.d, self.tol, self.theta = d, tol, theta
        self.max_sweeps = max_sweeps if max_sweeps > 0 else 10**7
        self.F = np.zeros(self.n_local + self.n_ghost)
        self.F[: self.n_local] = (1 - d) / self.n_global
        self.H = np.zeros(self.n_local)
        self.leak = 0.0
        self.sweeps = 0
        self.edges = 0
        self.done = False
        self.reduce(count=False)

    def reduce(self, count=True):
        a = np.abs(self.F[: self.n_local])
        self.stats[0] = float(a.sum())
        self.stats[1] = float(a.max()) if len(a) else 0.0
        self.stats[2] = self.leak
        if count:
            self.sweeps += 1

    def control(self):
        if self.done:
            return
        g = self.gathered.view(self.world, 4).numpy()
        r, fm = float(g[:, 0].sum()), float(g[:, 1].max())
        self.resid = r
        self.T = min(self.theta * r / self.n_global, fm)
        self.done = r <= self.tol or self.sweeps >= self.max_sweeps

    def sweep(self):
        if self.done:
            self.send.zero_()
            return
        f = self.F[: self.n_local].copy()
        sel = (f != 0) & (np.abs(f) >= self.T)
        fs = np.where(sel, f, 0.0)
        self.H += fs
        self.F[: self.n_local][sel] = 0.0
        self.leak += float(fs[self.deg == 0].sum())
        self.edges += int(self.deg[sel].sum())
        np.add.at(self.F, self.slot, self.d * fs[self.src] * self.p)
        self.send[: self.n_ghost] = torch.from_numpy(self.F[self.n_local:].copy())
        self.F[self.n_local:] = 0.0

    def heavy_local(self):
        pass                                         # the frontier sweep has no heavy gather

    def apply(self):
        if self.done:
            return
        off = 0
        recv = self.recv.numpy()
        for c in self.recv_counts:
            self.F[self.recv_idx[off:off + c]] += recv[off:off + c]
            off += c

    def poll(self):
        return self.done

    def global_residual(self):
        return float(self.gathered.view(self.world, 4)[:, 0].sum())

    def finish(self, tol, **_):
        return torch.from_numpy(self.H.copy()), {"residual_l1": self.resid, "sweeps": self.sweeps,
                                                  "diffused_edges": self.edges, "leak": self.leak}
