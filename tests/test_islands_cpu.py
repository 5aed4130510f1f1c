"""Island model host logic (paper_2504_00987_b200/islands.py) on CPU with the
gloo backend at world_size 2: elite all_gather, best-key all_reduce and stop
propagation. The solver is a deterministic stand-in with the labs_solver
surface; the device side of export/import is covered by the GPU tests."""
import ctypes as C
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


class FakeSolver:
    def __init__(self, rank, R, n, start, rate):
        self.rank, self.R, self.n, self.nw = rank, R, n, (n + 63) // 64
        self.best = np.array([start + 3 * r for r in range(R)], dtype=np.int64)
        self.rate, self.stopped, self.imports, self.epochs = rate, False, [], 0

    def run(self, epoch_seconds=-1.0, race=True):
        if not self.stopped:
            self.best = np.maximum(self.best - self.rate, 1)
            self.epochs += 1

    def status(self):
        r = int(np.argmin(self.best))
        return {"running": 0 if self.stopped else self.R,
                "best_energy": int(self.best[r]), "best_replica": self.rank * self.R + r}

    def export_elites(self, k, pw, pe):
        order = np.argsort(self.best, kind="stable")[:k]
        w = np.zeros(k * self.nw, dtype=np.int64)
        e = self.best[order].astype(np.int64)
        for i, r in enumerate(order):
            w[i * self.nw] = self.rank * 1000 + int(r)  # tag: origin rank/replica
        C.memmove(pw, w.ctypes.data, w.nbytes)
        C.memmove(pe, e.ctypes.data, e.nbytes)

    def import_elites(self, count, pw, pe, rotation=0):
        w = np.zeros(count * self.nw, dtype=np.int64)
        e = np.zeros(count, dtype=np.int64)
        C.memmove(w.ctypes.data, pw, w.nbytes)
        C.memmove(e.ctypes.data, pe, e.nbytes)
        self.imports.append((w[::self.nw].tolist(), e.tolist(), rotation))

    def request_stop(self):
        self.stopped = True

    def sync(self):
        pass


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2504_00987_b200.islands import Islands
    # rank 1 descends faster: it reaches the target first and must stop rank 0
    s = FakeSolver(rank, R=4, n=64, start=400 + 50 * rank, rate=10 + 15 * rank)
    isl = Islands(s, n=64, k_elites=2)
    rep = isl.run(target=208, epoch_seconds=0.0, exchange_every=2)
    q.put((rank, rep.best_energy, rep.best_replica, rep.reached, rep.epochs, rep.exchanges,
           s.stopped, s.imports[0] if s.imports else None))
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def test_islands_two_ranks_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    r0, r1 = out
    # same decision on both ranks: global best key, reached, epoch count
    assert r0[1:6] == r1[1:6]
    best_e, best_rep, reached, epochs, exchanges = r0[1:6]
    assert reached and best_e <= 208
    assert best_rep // 4 == 1  # rank 1's replica holds the lowest key
    assert exchanges == epochs // 2
    assert r0[6] and r1[6]  # both solvers told to stop
    # first exchange: each rank received both ranks' top-2 elites, rank order
    tags, energies, rot = r0[7]
    assert len(tags) == 4 and {t // 1000 for t in tags} == {0, 1}
    assert energies[:2] == sorted(energies[:2]) and energies[2:] == sorted(energies[2:])
    assert rot == 2
